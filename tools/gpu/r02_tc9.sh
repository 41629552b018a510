export PYTHONUNBUFFERED=1
RSH_TC_FLAGS=5 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_spmm_tc --launch-skip 3 --launch-count 1 -o gpurun_out/tc9_knob5 python tools/tc_probe.py stencil2m > gpurun_out/tc9_ncu.log 2>&1
tail -1 gpurun_out/tc9_ncu.log
