timeout 600 python -m pytest tests/test_reorder.py -q --tb=short 2>&1 | grep -v "^  \|^$" | tail -8
timeout 900 python tools/reorder_probe.py --workload rmat1m --hub-cap 256 2>&1 | tail -3
timeout 1500 python tools/reorder_probe.py --workload heavytail4m --hub-cap 256 2>&1 | tail -3
