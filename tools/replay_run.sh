# GPU: replay the BASELINE workloads' column sequences as pure B-row gathers (tools/microbench/replay_gather.cu)
# beside the streaming kernel's own time (tools/cc_probe.py).  Output under gpurun_out/.
set -x
mkdir -p gpurun_out
cd tools/microbench && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/replay_gather replay_gather.cu && cd ../..
for w in ${REPLAY_WORKLOADS:-rmat1m stencil2m heavytail4m}; do
  args=$(python tools/replay_dump.py $w /tmp/$w.cols)
  echo "== $w ($args)"
  timeout 300 /tmp/replay_gather /tmp/$w.cols $args
done > gpurun_out/replay.txt 2>&1
[ -n "$REPLAY_NO_PROBE" ] || timeout 600 python tools/cc_probe.py rmat1m stencil2m heavytail4m 0 > gpurun_out/replay_ccprobe.txt 2>&1
