export PYTHONUNBUFFERED=1
timeout 300 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -2
TC_KNOBS=5,256,512,768,1024,1280,261,517,773,1029,1285 timeout 600 python tools/tc_probe.py stencil2m 2>&1 | tee gpurun_out/tc13_probe.txt
