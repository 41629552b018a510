set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 ./tools/microbench/gather_plateau_bin 2>&1 | tee gpurun_out/r02_gather_plateau.txt
timeout 900 python tools/panel_probe.py rmat1m heavytail4m 2>&1 | tee gpurun_out/r02_panel_probe.txt
