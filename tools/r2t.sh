timeout 600 python tools/sanitize_cases.py c1 c5 prune passes split 2>&1 | tail -6
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 300 -p no:cacheprovider -k "random_small or configs_scaled or batch_sizes or counters or row_order or split or tile_passes or edge or empty or deterministic or resume" 2>&1 | tail -3
python tools/ab.py --config C5 --reps 2 --queries 2 ab_libs/E.so ab_libs/S.so
python tools/ab.py --config C3 --reps 2 --queries 2 ab_libs/E.so ab_libs/S.so
python tools/ab.py --config C1 --reps 3 --queries 5 ab_libs/E.so ab_libs/S.so
