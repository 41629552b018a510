timeout 600 python -m pytest tests/test_rst_io.py -x -q -m gpu 2>&1 | grep -v "^  " | tail -30
for v in 0 512 8 520; do echo "stencil v=$v"; timeout 300 python tools/probe_config.py --workload stencil2m --math fp32 --ccv $v --iters 20 2>&1 | grep spmm; done
timeout 300 python tools/probe_config.py --workload stencil2m --math fp32 --ccv 0 --iters 3 --check 2>&1 | tail -1
timeout 300 python tools/probe_config.py --workload uniform4k --math fp32 --ccv 0 --iters 20 --check 2>&1 | grep "spmm\|max_rel"
timeout 300 python tools/probe_config.py --workload uniform4k --math fp32 --ccv 512 --iters 20 2>&1 | grep "spmm\|max_rel"
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmm_stream -s 3 -c 1 -o gpurun_out/prof_stencil_slot python tools/probe_config.py --workload stencil2m --math fp32 --ccv 0 --iters 1 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/prof_stencil_slot.ncu-rep > gpurun_out/prof_stencil_slot.txt 2>&1
