export PYTHONUNBUFFERED=1
timeout 300 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -3
TC_KNOBS=1,4,5,261,1029 timeout 600 python tools/tc_probe.py stencil2m rmat1m heavytail4m 2>&1 | tee gpurun_out/tc8_probe.txt
