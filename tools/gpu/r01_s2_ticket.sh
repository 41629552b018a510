timeout 900 python -m pytest tests -q -m gpu -x --tb=short 2>&1 | grep -v "^  \|^$" | tail -4
for w in rmat1m heavytail4m; do echo "$w"; timeout 300 python tools/probe_config.py --workload $w --iters 30 2>&1 | grep spmm; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_spmm|k_fixup" -c 30 --csv --log-file gpurun_out/launches_rmat1m_timed.csv python bench.py --steps 8 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
grep "k_spmm\|k_fixup" gpurun_out/launches_rmat1m_timed.csv | head -6 | awk -F'","' '{print $5, $NF}'
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmm_stream -s 8 -c 1 -o gpurun_out/prof_heavy python bench.py --workload heavytail4m --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/prof_heavy.ncu-rep > gpurun_out/prof_heavy.txt 2>&1
rm -f gpurun_out/prof_heavy.ncu-rep
