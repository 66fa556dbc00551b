timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 300 -p no:cacheprovider -k "random_small or configs_scaled or head_feature or batch_sizes or multi_chunk or counters or layout" 2>&1 | tail -2
python tools/ab.py --config C4 --reps 2 --queries 1 ab_libs/E.so ab_libs/H64.so:32:0.125 ab_libs/H64.so:48:0.03125 ab_libs/H64.so
python tools/ab.py --config C2 --reps 3 --queries 4 ab_libs/E.so ab_libs/H64.so:32:0.125 ab_libs/H64.so:48:0.03125 ab_libs/H64.so
