for c in C2; do timeout 600 python tools/ab.py --config $c --reps 2 paper_1011_2807_b200/libknnjoin.so ab_libs/ld2.so 2>&1 | tail -2; done
timeout 600 python tools/ab.py --config C4 --rows-r 20000 --rows-s 2000000 --reps 1 paper_1011_2807_b200/libknnjoin.so ab_libs/ld2.so 2>&1 | tail -2
KREGEX='k_accumulate_topk<\(int\)2, \(int\)\d, \(bool\)\d, \(int\)8, \(bool\)1, \(bool\)0>' bash tools/runs/prof.sh r3j paper_1011_2807_b200/libknnjoin.so "C4 --rows-r 20000 --rows-s 2000000"
