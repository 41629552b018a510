./tools/microbench/bulk_gather_bin 2>&1 | tee gpurun_out/bulk_gather_microbench.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_spmm|k_fixup" -c 40 --csv --log-file gpurun_out/launches_rmat1m_timed.csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
tail -5 gpurun_out/launches_rmat1m_timed.csv
