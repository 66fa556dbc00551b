bash tools/runs/prof.sh r3c paper_1011_2807_b200/libknnjoin.so "C5 --rows-r 4000" "C3 --rows-r 10000"
