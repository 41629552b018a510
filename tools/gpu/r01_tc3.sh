./tools/microbench/umma_issue_bin | tee gpurun_out/umma_issue_v2.txt
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -4
for m in tf32 fp32; do timeout 300 python tools/probe_config.py --workload rmat1m --math $m --l1 1 --check 2>&1 | grep -E "spmm|max_rel|Error|error" ; done
timeout 300 python tools/probe_config.py --workload rmat1m --math tf32 --l1 0 2>&1 | grep -E "spmm|Error|error"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmm -s 2 -c 1 -o gpurun_out/prof_tc_r01c python tools/probe_config.py --workload rmat1m --math tf32 --iters 1 > gpurun_out/ncu_tc.log 2>&1; tail -1 gpurun_out/ncu_tc.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmm -s 2 -c 1 -o gpurun_out/prof_cc_r01c python tools/probe_config.py --workload rmat1m --math fp32 --iters 1 > gpurun_out/ncu_cc.log 2>&1; tail -1 gpurun_out/ncu_cc.log
