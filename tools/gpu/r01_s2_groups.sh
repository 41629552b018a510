timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "bit_identical or feature_widths or half_precision" --tb=short 2>&1 | grep -v "^  \|^$" | tail -8
for v in 0 2048; do echo "stencil v=$v"; timeout 300 python tools/probe_config.py --workload stencil2m --ccv $v --iters 20 2>&1 | grep spmm; done
timeout 300 python tools/probe_config.py --workload stencil2m --iters 3 --check 2>&1 | tail -1
for v in 0 2048; do echo "uniform v=$v"; timeout 300 python tools/probe_config.py --workload uniform4k --ccv $v --iters 50 2>&1 | grep spmm; done
for v in 0 1024; do echo "rmat v=$v"; timeout 300 python tools/probe_config.py --workload rmat1m --ccv $v --iters 20 2>&1 | grep spmm; done
for v in 0 1024; do echo "heavy v=$v"; timeout 300 python tools/probe_config.py --workload heavytail4m --ccv $v --iters 10 2>&1 | grep spmm; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmm_stream -s 3 -c 1 -o gpurun_out/prof_stream_stencil_g2 python tools/probe_config.py --workload stencil2m --iters 1 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/prof_stream_stencil_g2.ncu-rep > gpurun_out/prof_stream_stencil_g2.txt 2>&1
rm -f gpurun_out/prof_stream_stencil_g2.ncu-rep
