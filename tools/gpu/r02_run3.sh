export PYTHONUNBUFFERED=1
timeout 2400 python -m pytest tests -x -q -m gpu 2>&1 | tail -5 > gpurun_out/r02_pytest_gpu3.txt; cat gpurun_out/r02_pytest_gpu3.txt
timeout 600 python bench.py --workload stencil2m --steps 20 --warmup 5 --no-ncu > gpurun_out/r02_bench_stencil2m.json 2> gpurun_out/r02_bench_stencil2m.err; tail -2 gpurun_out/r02_bench_stencil2m.err
python -c "import json;d=json.load(open('gpurun_out/r02_bench_stencil2m.json'));print(d['value'],d['ms_per_step'],d['dtype'],d['details']['path_ms'],d['roofline']['frac'])"
