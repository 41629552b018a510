set -x
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -15
for m in tf32 fp32; do for l in 1 0; do timeout 300 python tools/probe_config.py --workload rmat1m --math $m --l1 $l --check 2>&1 | grep -E "spmm|max_rel|Error|error" ; done; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmm_tc -s 2 -c 1 -o gpurun_out/prof_tc_r01b python tools/probe_config.py --workload rmat1m --math tf32 --iters 1 > gpurun_out/ncu_tc.log 2>&1; tail -2 gpurun_out/ncu_tc.log
