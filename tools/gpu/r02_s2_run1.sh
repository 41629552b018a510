set -x
export PYTHONUNBUFFERED=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_rmat1m.json 2> gpurun_out/r02_bench_rmat1m.err; tail -3 gpurun_out/r02_bench_rmat1m.err
cat gpurun_out/r02_bench_rmat1m.json
timeout 600 ./tools/microbench/gather_plateau_bin > gpurun_out/r02_gather_plateau.txt 2>&1
timeout 900 python tools/panel_probe.py rmat1m heavytail4m > gpurun_out/r02_panel_probe.txt 2>&1
timeout 3000 python -m pytest tests -x -q -m gpu --durations=15 > gpurun_out/r02_pytest_gpu.txt 2>&1
tail -25 gpurun_out/r02_pytest_gpu.txt
