for l in 1 0 4 5 8 12; do timeout 120 python tools/probe_config.py --workload rmat1m --math tf32 --l1 $l 2>&1 | grep -E "spmm|Error|error"; done
timeout 120 python tools/probe_config.py --workload rmat1m --math fp32 --check 2>&1 | grep -E "spmm|max_rel|Error|error"
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
