bash tools/runs/prof.sh r3d paper_1011_2807_b200/libknnjoin.so "C3 --rows-r 10000"
