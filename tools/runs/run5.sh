timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/r3b_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r3b_pytest.log
for c in C5 C3 C1; do timeout 600 python tools/ab.py --config $c --reps 2 ab_libs/base.so paper_1011_2807_b200/libknnjoin.so 2>&1 | tail -2; done
