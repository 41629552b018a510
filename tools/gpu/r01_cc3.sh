for v in 0 1 2 3; do timeout 120 python tools/probe_config.py --workload rmat1m --math fp32 --ccv $v --check 2>&1 | grep -E "spmm|max_rel|Error|error"; done
for w in stencil2m heavytail4m; do timeout 300 python tools/probe_config.py --workload $w --math fp32 2>&1 | grep -E "spmm|Error|error"; done
timeout 300 python tools/probe_config.py --workload heavytail4m --math auto 2>&1 | grep -E "spmm|Error|error"
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
