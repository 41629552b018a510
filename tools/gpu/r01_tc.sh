set -x
./tools/microbench/umma_probe_bin 2>&1 | tee gpurun_out/umma_probe_v2.txt
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -25
for m in fp32 tf32; do for l in 1 0; do timeout 300 python tools/probe_config.py --workload rmat1m --math $m --l1 $l --check 2>&1 | grep -E "spmm|max_rel|Error|error" ; done; done
