set -x
for v in 0 128 8 136 64; do timeout 300 python tools/probe_config.py --workload rmat1m --math fp32 --ccv $v --iters 20 2>&1 | grep spmm; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmm -s 3 -c 1 -o gpurun_out/prof_stream_v0 python tools/probe_config.py --workload rmat1m --math fp32 --ccv 0 --iters 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmm -s 3 -c 1 -o gpurun_out/prof_legacy python tools/probe_config.py --workload rmat1m --math fp32 --ccv 64 --iters 1 > /dev/null 2>&1
ls -la gpurun_out
