bash tools/runs/prof.sh r3new paper_1011_2807_b200/libknnjoin.so "C5 --rows-r 4000" "C3 --rows-r 10000"
bash tools/runs/prof.sh r3base ab_libs/base.so "C5 --rows-r 4000"
