set -x
python -m pytest tests -x -q -m gpu 2>&1 | tail -15
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
python bench.py --steps 50 --warmup 5 > gpurun_out/bench_s2a.json 2> gpurun_out/bench_s2a.err; tail -3 gpurun_out/bench_s2a.err; cat gpurun_out/bench_s2a.json
