python bench.py --steps 200 --warmup 5 > gpurun_out/bench_r01b.json 2> gpurun_out/bench_r01b.err; tail -3 gpurun_out/bench_r01b.err; cat gpurun_out/bench_r01b.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches_r01b.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 --math fp32 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmm_cc -s 8 -c 1 -o gpurun_out/prof_cc_r01h python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --math fp32 > gpurun_out/ncu_full.log 2>&1; tail -1 gpurun_out/ncu_full.log
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_r01b.json 2>&1; tail -1 gpurun_out/bench_ref_r01b.json
