# full GPU suite on the current code, then compute-sanitizer (T9) over tools/sanitize_cases.py
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/r2s_pytest.log 2>&1; echo pytest rc=$?
grep -E "passed|failed|FAILED" gpurun_out/r2s_pytest.log | tail -15
timeout 300 python tools/sanitize_cases.py > gpurun_out/r2s_plain.log 2>&1; echo plain rc=$?; tail -3 gpurun_out/r2s_plain.log
for tool in memcheck synccheck initcheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 python tools/sanitize_cases.py > gpurun_out/r2s_$tool.log 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/r2s_$tool.log
done
