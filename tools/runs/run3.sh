L=paper_1011_2807_b200/libknnjoin.so
timeout 900 python tools/ab.py --config C5 --rows-r 4000 --reps 2 $L $L:tiles_per_pass=1 $L:tiles_per_pass=4 $L:tiles_per_pass=8 $L:tiles_per_pass=62 ab_libs/base.so:tiles_per_pass=1 2>&1 | tail -6
timeout 900 python tools/ab.py --config C3 --rows-r 10000 --reps 2 $L $L:tiles_per_pass=1 $L:tiles_per_pass=4 $L:tiles_per_pass=16 $L:tiles_per_pass=123 2>&1 | tail -5
