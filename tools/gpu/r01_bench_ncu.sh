set -x
./tools/microbench/umma_probe_bin 2>&1 | tee gpurun_out/umma_probe.txt
python -m pytest tests -x -q -m gpu 2>&1 | tail -5
python bench.py --steps 100 --warmup 5 > gpurun_out/bench_r01a.json 2> gpurun_out/bench_r01a.err; tail -3 gpurun_out/bench_r01a.err; cat gpurun_out/bench_r01a.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_r01a.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_spmm_cc -s 3 -c 1 -o gpurun_out/prof_spmm_r01a python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_full.log 2>&1; tail -3 gpurun_out/ncu_full.log
ls -la gpurun_out
