export PYTHONUNBUFFERED=1
TC_KNOBS=1 timeout 600 python tools/tc_probe.py stencil2m 2>&1 | tee gpurun_out/tc3_probe.txt
