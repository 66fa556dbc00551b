L=paper_1011_2807_b200/libknnjoin.so
timeout 900 python tools/ab.py --config C5 --rows-r 4000 --reps 2 $L $L:tile=12288 $L:tile=14336 $L:tile=6144 2>&1 | tail -4
timeout 900 python tools/ab.py --config C3 --rows-r 10000 --reps 2 $L $L:tile=12288 $L:tile=14336 $L:tile=6144 2>&1 | tail -4
