for w in rmat1m heavytail4m; do for e in 0 1; do echo "$w no_lpt=$e"; if [ $e = 1 ]; then export RSH_NO_LPT=1; else unset RSH_NO_LPT; fi; timeout 300 python tools/probe_config.py --workload $w --iters 30 2>&1 | grep spmm; done; done
unset RSH_NO_LPT
timeout 900 python -m pytest tests -q -m gpu -x --tb=short 2>&1 | grep -v "^  \|^$" | tail -3
