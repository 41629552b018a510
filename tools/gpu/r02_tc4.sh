export PYTHONUNBUFFERED=1
RSH_TC_FLAGS=7 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_spmm_tc --launch-skip 3 --launch-count 1 -o gpurun_out/tc4_knob7 python tools/tc_probe.py stencil2m > gpurun_out/tc4_ncu.log 2>&1
tail -2 gpurun_out/tc4_ncu.log
