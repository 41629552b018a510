export PYTHONUNBUFFERED=1
TC_KNOBS=5,37,32,33,36 timeout 600 python tools/tc_probe.py stencil2m rmat1m 2>&1 | tee gpurun_out/tc14_probe.txt
