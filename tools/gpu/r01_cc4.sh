timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for v in 0 3; do timeout 120 python tools/probe_config.py --workload rmat1m --math fp32 --ccv $v 2>&1 | grep -E "spmm|Error|error"; done
timeout 300 python tools/probe_config.py --workload heavytail4m --math fp32 2>&1 | grep -E "spmm|Error|error"
timeout 300 python tools/probe_config.py --workload heavytail4m --math auto 2>&1 | grep -E "spmm|Error|error"
timeout 120 python tools/probe_config.py --workload rmat1m --math tf32 2>&1 | grep -E "spmm|Error|error"
