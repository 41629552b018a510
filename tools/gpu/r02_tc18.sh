export PYTHONUNBUFFERED=1
TC_KNOBS=0,256,512,768,1024,1280 timeout 600 python tools/tc_probe.py stencil2m 2>&1 | tee gpurun_out/tc18_probe.txt
