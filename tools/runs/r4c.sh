#!/bin/bash
# T9 on the final code: checked build (-DKJ_CHECKS bounds checks + KNNJOIN_MAX_CTAS schedules) over the sanitize
# cases and the parity / precision / prune / iiib suites
mkdir -p gpurun_out
KNNJOIN_LIB=ab_libs/checked/libknnjoin.so timeout 900 python tools/sanitize_cases.py > gpurun_out/r4c_checked_cases.log 2>&1; echo checked rc=$?; tail -12 gpurun_out/r4c_checked_cases.log
KNNJOIN_LIB=ab_libs/checked/libknnjoin.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_precision.py tests/test_gpu_prune.py tests/test_gpu_iiib.py -m gpu -q -x --timeout 600 -p no:cacheprovider -k "not full_size and not every_row" > gpurun_out/r4c_checked_pytest.log 2>&1; echo checked-pytest rc=$?; tail -3 gpurun_out/r4c_checked_pytest.log
timeout 900 python -m pytest tests/test_gpu_checks.py -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/r4c_checks.log 2>&1; echo checks rc=$?; tail -3 gpurun_out/r4c_checks.log
