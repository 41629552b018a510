timeout 900 python -m pytest tests -q -m gpu -x --tb=short 2>&1 | grep -v "^  \|^$" | tail -4
for w in rmat1m heavytail4m stencil2m; do echo "$w"; timeout 300 python tools/probe_config.py --workload $w --iters 30 2>&1 | grep spmm; done
timeout 300 python tools/probe_config.py --workload heavytail4m --iters 2 --check 2>&1 | tail -1
