./tools/microbench/gather_bw2_bin | tee gpurun_out/gather_bw2.txt
timeout 120 python tools/tc_profile.py --flags 5
