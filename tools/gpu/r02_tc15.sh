export PYTHONUNBUFFERED=1
TC_KNOBS=37,101,165,36,100,164,0,128 timeout 600 python tools/tc_probe.py stencil2m 2>&1 | tee gpurun_out/tc15_probe.txt
