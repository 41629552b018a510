timeout 900 python -m pytest tests -q -m gpu -x --tb=short 2>&1 | grep -v "^  \|^$" | tail -6
for w in rmat1m stencil2m heavytail4m uniform4k; do for v in 0 4096; do echo "$w v=$v"; timeout 300 python tools/probe_config.py --workload $w --ccv $v --iters 20 2>&1 | grep spmm; done; done
timeout 300 python tools/probe_config.py --workload heavytail4m --iters 2 --check 2>&1 | tail -1
