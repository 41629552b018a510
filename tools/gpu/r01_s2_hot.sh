for v in 0 128; do echo "rmat v=$v"; timeout 300 python tools/probe_config.py --workload rmat1m --math fp32 --ccv $v --iters 20 2>&1 | grep spmm; done
for bud in 33554432 100663296; do echo "rmat budget=$bud"; RSH_HOT_BUDGET=$bud timeout 300 python tools/probe_config.py --workload rmat1m --math fp32 --ccv 0 --iters 20 2>&1 | grep spmm; done
for v in 0 128; do echo "heavy v=$v"; timeout 300 python tools/probe_config.py --workload heavytail4m --ccv $v --iters 10 2>&1 | grep spmm; done
for v in 0 128; do echo "stencil v=$v"; timeout 300 python tools/probe_config.py --workload stencil2m --ccv $v --iters 20 2>&1 | grep spmm; done
timeout 300 python tools/probe_config.py --workload rmat1m --math fp32 --iters 3 --check 2>&1 | tail -1
timeout 900 python -m pytest tests -q -m gpu --tb=short 2>&1 | grep -v "^  \|^$" | tail -40
