export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_api.py -x -q 2>&1 | tail -3
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_run.py > gpurun_out/r02_sanitizer_$tool.txt 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/r02_sanitizer_$tool.txt
done
