export PYTHONUNBUFFERED=1
TC_KNOBS=109,2157,4205,0,2048,4096 timeout 600 python tools/tc_probe.py stencil2m rmat1m 2>&1 | tee gpurun_out/tc17_probe.txt
