export PYTHONUNBUFFERED=1
TC_KNOBS=101,109 timeout 600 python tools/tc_probe.py stencil2m 2>&1 | tee gpurun_out/tc16_probe.txt
RSH_TC_FLAGS=109 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_spmm_tc --launch-skip 3 --launch-count 1 -o gpurun_out/tc16_k109 python tools/tc_probe.py stencil2m > gpurun_out/tc16_ncu.log 2>&1
