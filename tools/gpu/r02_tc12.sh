export PYTHONUNBUFFERED=1
RSH_TC_FLAGS=5 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_spmm_tc --launch-skip 3 --launch-count 1 -o gpurun_out/tc12_knob5 python tools/tc_probe.py stencil2m > gpurun_out/tc12_ncu.log 2>&1
RSH_TC_FLAGS=0 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_spmm_tc --launch-skip 3 --launch-count 1 -o gpurun_out/tc12_full python tools/tc_probe.py stencil2m > gpurun_out/tc12b_ncu.log 2>&1
tail -1 gpurun_out/tc12_ncu.log gpurun_out/tc12b_ncu.log
