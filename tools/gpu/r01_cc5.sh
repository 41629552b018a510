for v in 0 3 4 7; do timeout 120 python tools/probe_config.py --workload rmat1m --math fp32 --ccv $v 2>&1 | grep -E "spmm|Error|error"; done
timeout 120 python tools/probe_config.py --workload rmat1m --math fp32 --check 2>&1 | grep -E "max_rel|Error|error"
timeout 300 python tools/probe_config.py --workload heavytail4m --math fp32 2>&1 | grep -E "spmm|Error|error"
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
