set -x
for v in 64 72 80 88 200; do timeout 300 python tools/probe_config.py --workload rmat1m --math fp32 --ccv $v --iters 20 2>&1 | grep spmm; done
timeout 300 python tools/probe_config.py --workload rmat1m --math fp32 --ccv 72 --iters 3 --check 2>&1 | tail -1
for v in 64 72 80; do timeout 300 python tools/probe_config.py --workload stencil2m --math fp32 --ccv $v --iters 20 2>&1 | grep spmm; done
for v in 64 72 80; do timeout 300 python tools/probe_config.py --workload heavytail4m --math fp32 --ccv $v --iters 10 2>&1 | grep spmm; done
RSH_CC_VARIANT=72 timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmm -s 3 -c 1 -o gpurun_out/prof_stream_v3 python tools/probe_config.py --workload rmat1m --math fp32 --ccv 72 --iters 1 > /dev/null 2>&1
