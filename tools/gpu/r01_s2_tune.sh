for w in rmat1m heavytail4m stencil2m; do for v in 0 8 24 48; do echo "$w v=$v"; timeout 300 python tools/probe_config.py --workload $w --ccv $v --iters 20 2>&1 | grep spmm; done; done
