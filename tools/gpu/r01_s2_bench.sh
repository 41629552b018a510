timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_rmat1m.json 2> gpurun_out/bench_rmat1m.err; tail -2 gpurun_out/bench_rmat1m.err; cat gpurun_out/bench_rmat1m.json
for w in uniform4k stencil2m heavytail4m; do timeout 900 python bench.py --workload $w --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; tail -1 gpurun_out/bench_$w.err; cat gpurun_out/bench_$w.json; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/launches_rmat1m_s2.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmm_stream -s 8 -c 1 -o gpurun_out/prof_bench_rmat1m_s2 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmm_stream -s 8 -c 1 -o gpurun_out/prof_bench_stencil2m_s2 python bench.py --workload stencil2m --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
ls gpurun_out
