timeout 900 python -m pytest tests -q -m gpu --tb=short 2>&1 | grep -v "^  \|^$" | tail -8
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_rmat1m.json 2> gpurun_out/bench_rmat1m.err; tail -2 gpurun_out/bench_rmat1m.err; cat gpurun_out/bench_rmat1m.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_rmat1m.json 2>&1; tail -1 gpurun_out/bench_ref_rmat1m.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/launches_rmat1m_s2.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmm_stream -s 8 -c 1 -o gpurun_out/prof_bench_rmat1m_s2 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/prof_bench_rmat1m_s2.ncu-rep > gpurun_out/prof_bench_rmat1m_s2.txt 2>&1
ncu -i gpurun_out/prof_bench_rmat1m_s2.ncu-rep --page source --csv --print-source sass > gpurun_out/sass_rmat1m_s2.csv 2>/dev/null
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --workload rmat16m --sharded --steps 10 --warmup 3 > gpurun_out/bench_rmat16m_n1.json 2> gpurun_out/bench_rmat16m_n1.err; tail -3 gpurun_out/bench_rmat16m_n1.err; cat gpurun_out/bench_rmat16m_n1.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 1 --sharded --steps 20 --warmup 3 > gpurun_out/bench_rmat1m_sharded_n1.json 2> gpurun_out/bench_rmat1m_sharded_n1.err; tail -3 gpurun_out/bench_rmat1m_sharded_n1.err; cat gpurun_out/bench_rmat1m_sharded_n1.json
du -sh gpurun_out/*
