timeout 300 python tools/probe_config.py --workload stencil2m --math fp32 --check 2>&1 | grep -E "spmm|max_rel|Error|error"
timeout 120 python tools/probe_config.py --workload uniform4k --math fp32 --check 2>&1 | grep -E "spmm|max_rel|Error|error"
for w in uniform4k rmat1m stencil2m heavytail4m; do python bench.py --workload $w --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_r01_$w.json 2> gpurun_out/bench_r01_$w.err; tail -c 600 gpurun_out/bench_r01_$w.json; echo; done
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
