timeout 120 python tools/tc_profile.py --flags 1
for l in 1 0; do timeout 120 python tools/probe_config.py --workload rmat1m --math tf32 --l1 $l --check 2>&1 | grep -E "spmm|max_rel|Error|error"; done
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
