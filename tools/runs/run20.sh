timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/r3n_pytest.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/r3n_pytest.log
L=paper_1011_2807_b200/libknnjoin.so
timeout 600 python tools/ab.py --config C2 --reps 2 ab_libs/v5.so $L $L:head_max=64,head_density=0.03125 $L:head_max=48,head_density=0.03125 2>&1 | tail -4
timeout 900 python tools/ab.py --config C4 --rows-r 20000 --rows-s 2000000 --reps 1 ab_libs/v5.so $L $L:head_max=64,head_density=0.03125 $L:head_max=48,head_density=0.03125 $L:head_max=64,head_density=0.02 2>&1 | tail -5
