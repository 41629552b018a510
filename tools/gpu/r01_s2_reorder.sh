timeout 600 python -m pytest tests/test_reorder.py -q --tb=short 2>&1 | grep -v "^  \|^$" | tail -20
timeout 900 python tools/reorder_probe.py --workload rmat1m --hub-cap 256 2>&1 | tail -4
timeout 900 python tools/reorder_probe.py --workload stencil2m --hub-cap 256 2>&1 | tail -4
timeout 1200 python tools/reorder_probe.py --workload heavytail4m --hub-cap 256 2>&1 | tail -4
