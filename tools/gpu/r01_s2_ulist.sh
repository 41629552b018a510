timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x --tb=short 2>&1 | grep -v "^  \|^$" | tail -6
for w in rmat1m stencil2m heavytail4m uniform4k; do for v in 0 4096; do echo "$w v=$v"; timeout 300 python tools/probe_config.py --workload $w --ccv $v --iters 20 2>&1 | grep spmm; done; done
timeout 300 python tools/probe_config.py --workload stencil2m --iters 3 --check 2>&1 | tail -1
