timeout 120 python tools/tc_profile.py --flags 1
timeout 120 python tools/tc_profile.py --flags 13
timeout 120 python tools/probe_config.py --workload rmat1m --math tf32 --l1 1 --check 2>&1 | grep -E "spmm|max_rel|Error|error"
