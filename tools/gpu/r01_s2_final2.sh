timeout 900 python -m pytest tests -q -m gpu --tb=short 2>&1 | grep -v "^  \|^$" | tail -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py --steps 100 --warmup 5 > gpurun_out/bench_rmat1m.json 2> gpurun_out/bench_rmat1m.err; tail -1 gpurun_out/bench_rmat1m.json
for w in uniform4k stencil2m heavytail4m; do timeout 900 python bench.py --workload $w --steps 50 --warmup 5 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; tail -1 gpurun_out/bench_$w.json; done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29513 bench.py --workload rmat16m --sharded --steps 10 --warmup 3 > gpurun_out/bench_rmat16m_n1.json 2> gpurun_out/bench_rmat16m_n1.err; cat gpurun_out/bench_rmat16m_n1.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_spmm|k_fixup" -c 30 --csv --log-file gpurun_out/launches_stencil2m_timed.csv python bench.py --workload stencil2m --steps 8 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
