timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/r3f_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r3f_pytest.log
for c in C5 C3 C2; do timeout 600 python tools/ab.py --config $c --reps 2 ab_libs/v3.so paper_1011_2807_b200/libknnjoin.so 2>&1 | tail -2; done
timeout 600 python tools/ab.py --config C4 --rows-r 20000 --rows-s 2000000 --reps 1 ab_libs/v3.so paper_1011_2807_b200/libknnjoin.so 2>&1 | tail -2
for c in C4 C5; do timeout 600 python bench.py --config $c --steps 2 --warmup 1 --no-e2e --no-cpu-baseline | python -c "import json,sys; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c build ms', j['breakdown']['build_index_ms'], 'K3', j['breakdown']['kernel_ms'])"; done
