for c in C2; do timeout 600 python tools/ab.py --config $c --reps 3 paper_1011_2807_b200/libknnjoin.so ab_libs/u2.so 2>&1 | tail -2; done
timeout 600 python tools/ab.py --config C4 --rows-r 20000 --rows-s 2000000 --reps 1 paper_1011_2807_b200/libknnjoin.so ab_libs/u2.so 2>&1 | tail -2
