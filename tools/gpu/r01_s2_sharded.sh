timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29514 bench.py --gpus 1 --sharded --steps 20 --warmup 3 > gpurun_out/bench_rmat1m_sharded_n1.json 2> gpurun_out/bench_rmat1m_sharded_n1.err; echo "stdout lines: $(wc -l < gpurun_out/bench_rmat1m_sharded_n1.json)"; cat gpurun_out/bench_rmat1m_sharded_n1.json; tail -3 gpurun_out/bench_rmat1m_sharded_n1.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmm_stream -s 3 -c 1 -o gpurun_out/prof_stencil python tools/probe_config.py --workload stencil2m --iters 1 > /dev/null 2>&1
ncu -i gpurun_out/prof_stencil.ncu-rep --page source --csv --print-source sass > gpurun_out/sass_stencil.csv 2>/dev/null
rm -f gpurun_out/prof_stencil.ncu-rep
