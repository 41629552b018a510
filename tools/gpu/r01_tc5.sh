timeout 120 python tools/probe_config.py --workload rmat1m --math tf32 --l1 1 --check 2>&1 | grep -E "spmm|max_rel|Error|error"
timeout 120 python tools/probe_config.py --workload rmat1m --math tf32 --l1 0 2>&1 | grep -E "spmm|Error|error"
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -4
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_spmm_tc -s 2 -c 1 -o gpurun_out/prof_tc_r01e python tools/probe_config.py --workload rmat1m --math tf32 --iters 1 > gpurun_out/ncu_tc.log 2>&1; tail -1 gpurun_out/ncu_tc.log
