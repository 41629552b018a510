export PYTHONUNBUFFERED=1
timeout 900 python tools/hot_probe.py rmat1m heavytail4m stencil2m 2>&1 | tee gpurun_out/r02_hot_probe.txt
