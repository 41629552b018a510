export PYTHONUNBUFFERED=1
timeout 300 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -15 > gpurun_out/tc1_pytest.txt
cat gpurun_out/tc1_pytest.txt
timeout 600 python tools/tc_probe.py stencil2m rmat1m uniform4k heavytail4m 2>&1 | tee gpurun_out/tc1_probe.txt
