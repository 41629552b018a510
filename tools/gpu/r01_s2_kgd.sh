for v in 0 8 24; do echo "stencil v=$v"; timeout 300 python tools/probe_config.py --workload stencil2m --ccv $v --iters 30 2>&1 | grep spmm; done
for v in 0 8 24; do echo "uniform v=$v"; timeout 300 python tools/probe_config.py --workload uniform4k --ccv $v --iters 50 2>&1 | grep spmm; done
