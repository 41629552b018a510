export PYTHONUNBUFFERED=1
timeout 300 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -15 > gpurun_out/tc2_pytest.txt
cat gpurun_out/tc2_pytest.txt
timeout 600 python tools/tc_probe.py stencil2m rmat1m 2>&1 | tee gpurun_out/tc2_probe.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_spmm_tc --launch-skip 3 --launch-count 1 -o gpurun_out/tc2_stencil python tools/tc_probe.py stencil2m > gpurun_out/tc2_ncu.log 2>&1
tail -3 gpurun_out/tc2_ncu.log
