mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_multilayer.py -m gpu -q -x -k "timeline or tiny" > gpurun_out/c9_pytest.log 2>&1; tail -3 gpurun_out/c9_pytest.log
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py > gpurun_out/c9_sanitizer_$tool.txt 2>&1
  echo "== $tool rc=$?"; tail -4 gpurun_out/c9_sanitizer_$tool.txt
done
