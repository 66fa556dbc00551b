timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/r3e_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r3e_pytest.log
for c in C5 C3; do timeout 600 python tools/ab.py --config $c --reps 2 ab_libs/base.so ab_libs/v2.so paper_1011_2807_b200/libknnjoin.so 2>&1 | tail -3; done
