timeout 900 python -m pytest tests -q -m gpu --tb=short 2>&1 | grep -v "^  \|^$" | tail -4
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py --steps 100 --warmup 5 > gpurun_out/bench_rmat1m.json 2> gpurun_out/bench_rmat1m.err; tail -1 gpurun_out/bench_rmat1m.json
for w in uniform4k stencil2m heavytail4m; do timeout 900 python bench.py --workload $w --steps 50 --warmup 5 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; tail -1 gpurun_out/bench_$w.json; done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29515 bench.py --workload rmat16m --sharded --steps 10 --warmup 3 > gpurun_out/bench_rmat16m_n1.json 2> gpurun_out/bench_rmat16m_n1.err; cat gpurun_out/bench_rmat16m_n1.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_rmat1m.json 2>&1; tail -1 gpurun_out/bench_ref_rmat1m.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_spmm|k_fixup" -c 30 --csv --log-file gpurun_out/launches_rmat1m_timed.csv python bench.py --steps 8 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmm_stream -s 8 -c 1 -o gpurun_out/prof_rmat1m python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/prof_rmat1m.ncu-rep > gpurun_out/prof_rmat1m.txt 2>&1
ncu -i gpurun_out/prof_rmat1m.ncu-rep --page source --csv --print-source sass > gpurun_out/sass_rmat1m.csv 2>/dev/null
rm -f gpurun_out/prof_rmat1m.ncu-rep
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmm_stream -s 8 -c 1 -o gpurun_out/prof_stencil python bench.py --workload stencil2m --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/prof_stencil.ncu-rep > gpurun_out/prof_stencil.txt 2>&1
rm -f gpurun_out/prof_stencil.ncu-rep
