set -x
python tools/smoke_debug.py 2>&1 | tail -8
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -6
for v in 0 8 16 24 32 64; do timeout 300 python tools/probe_config.py --workload rmat1m --math fp32 --ccv $v --iters 20 2>&1 | grep spmm; done
timeout 300 python tools/probe_config.py --workload rmat1m --math fp32 --ccv 0 --iters 5 --check 2>&1 | tail -2
for v in 0 16 64; do timeout 300 python tools/probe_config.py --workload stencil2m --math fp32 --ccv $v --iters 20 2>&1 | grep spmm; done
for v in 0 16; do timeout 300 python tools/probe_config.py --workload heavytail4m --math fp32 --ccv $v --iters 10 2>&1 | grep spmm; done
timeout 300 python tools/probe_config.py --workload heavytail4m --math auto --iters 10 2>&1 | grep spmm
