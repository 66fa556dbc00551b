timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/r3h_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r3h_pytest.log
for c in C5 C3 C2; do timeout 600 python tools/ab.py --config $c --reps 2 ab_libs/v3.so paper_1011_2807_b200/libknnjoin.so 2>&1 | tail -2; done
timeout 600 python tools/ab.py --config C4 --rows-r 20000 --rows-s 2000000 --reps 1 ab_libs/v3.so paper_1011_2807_b200/libknnjoin.so 2>&1 | tail -2
