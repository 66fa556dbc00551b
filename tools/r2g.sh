python tools/ab.py --config C4 --reps 2 --queries 1 ab_libs/E.so ab_libs/G.so
python tools/ab.py --config C2 --reps 3 --queries 4 ab_libs/E.so ab_libs/G.so
