export PYTHONUNBUFFERED=1
TC_KNOBS=0,16,7,15,23,31,3,19,4,20 timeout 600 python tools/tc_probe.py stencil2m 2>&1 | tee gpurun_out/tc5_probe.txt
