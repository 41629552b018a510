set -x
export PYTHONUNBUFFERED=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_rmat1m.json 2> gpurun_out/r02_bench_rmat1m.err; tail -3 gpurun_out/r02_bench_rmat1m.err
timeout 600 python tools/l2_probe.py rmat1m heavytail4m 2>&1 | tee gpurun_out/r02_l2_probe.txt
timeout 600 ./tools/microbench/gather_plateau_bin 2>&1 | tee gpurun_out/r02_gather_plateau2.txt
timeout 3000 python -m pytest tests -x -q -m gpu --durations=15 2>&1 | tail -40 > gpurun_out/r02_pytest_gpu.txt
tail -5 gpurun_out/r02_pytest_gpu.txt
