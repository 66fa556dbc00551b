timeout 900 python -m pytest tests/test_gpu_precision.py tests/test_gpu_iiib.py -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/r2c_pytest.log 2>&1; echo rc=$?
grep -E "passed|failed|FAILED|Error" gpurun_out/r2c_pytest.log | head -40
