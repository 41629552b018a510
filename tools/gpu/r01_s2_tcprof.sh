timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "bit_identical" --tb=short 2>&1 | grep -v "^  \|^$" | tail -8
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmm_tc -s 3 -c 1 -o gpurun_out/prof_tc_rmat1m python tools/probe_config.py --workload rmat1m --math tf32 --iters 1 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/prof_tc_rmat1m.ncu-rep > gpurun_out/prof_tc_rmat1m.txt 2>&1
rm -f gpurun_out/prof_tc_rmat1m.ncu-rep
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmm_stream -s 3 -c 1 -o gpurun_out/prof_stream_stencil python tools/probe_config.py --workload stencil2m --iters 1 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/prof_stream_stencil.ncu-rep > gpurun_out/prof_stream_stencil.txt 2>&1
rm -f gpurun_out/prof_stream_stencil.ncu-rep
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmm_stream -s 3 -c 1 -o gpurun_out/prof_stream_heavy python tools/probe_config.py --workload heavytail4m --iters 1 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/prof_stream_heavy.ncu-rep > gpurun_out/prof_stream_heavy.txt 2>&1
rm -f gpurun_out/prof_stream_heavy.ncu-rep
ls -la gpurun_out
