# GPU: the round's measurement set -- bench.py lines for BASELINE configs 1-5 (config 5 on the
# row-shard path under torchrun, N=1), the reference arm, the ncu launch list of the default run
# and one `ncu --set full` capture of the streaming kernel on config 2.  Output under gpurun_out/.
mkdir -p gpurun_out/rb
for w in uniform4k rmat1m stencil2m heavytail4m; do
  timeout 900 python bench.py --workload $w > gpurun_out/rb/bench_$w.json 2> gpurun_out/rb/bench_$w.err
done
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 \
  bench.py --sharded --workload rmat16m --steps 20 --warmup 3 > gpurun_out/rb/bench_rmat16m_sharded.json 2> gpurun_out/rb/bench_rmat16m.err
timeout 900 python bench.py --impl reference > gpurun_out/rb/bench_reference.json 2> gpurun_out/rb/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/rb/launches_rmat1m.csv \
  python bench.py --steps 3 --warmup 3 --no-ncu --no-cpu-baseline --e2e-steps 2 > gpurun_out/rb/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmm_stream --launch-skip 3 -c 1 -f -o gpurun_out/rb/stream_rmat1m \
  python bench.py --kernel-only --workload rmat1m > gpurun_out/rb/ncu_full.log 2>&1
python tools/ncu_summary.py gpurun_out/rb/stream_rmat1m.ncu-rep > gpurun_out/rb/ncu_stream_rmat1m.txt 2>&1
