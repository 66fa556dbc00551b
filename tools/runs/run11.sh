for c in C5 C3; do timeout 600 python tools/ab.py --config $c --reps 2 paper_1011_2807_b200/libknnjoin.so ab_libs/d2.so ab_libs/d4.so 2>&1 | tail -3; done
bash tools/runs/prof.sh r3g paper_1011_2807_b200/libknnjoin.so "C5 --rows-r 4000" "C3 --rows-r 10000"
