for v in 0 1 2 3; do timeout 120 python tools/probe_config.py --workload rmat1m --math fp32 --ccv $v --check 2>&1 | grep -E "spmm|max_rel|Error|error"; done
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_spmm_cc -s 2 -c 1 -o gpurun_out/prof_cc_r01g python tools/probe_config.py --workload rmat1m --math fp32 --iters 1 > gpurun_out/ncu_cc.log 2>&1; tail -1 gpurun_out/ncu_cc.log
