./tools/microbench/tma_gather_bin | tee gpurun_out/tma_gather.txt
timeout 120 python tools/probe_config.py --workload rmat1m --math fp32 2>&1 | grep -E "spmm|Error|error"
