#!/bin/bash
# session 3, call b: A/B of head-free exchange scan (xc) and block-path slice bounds one tile ahead (pf)
mkdir -p gpurun_out
V="ab_libs/base.so ab_libs/xc.so ab_libs/pf.so"
timeout 900 python tools/ab.py --config C4 --rows-r 20000 --rows-s 2000000 --reps 2 $V > gpurun_out/s3b_ab_C4s.txt 2>&1; echo "C4s rc=$?"; cat gpurun_out/s3b_ab_C4s.txt
timeout 600 python tools/ab.py --config C2 --reps 3 --queries 4 $V > gpurun_out/s3b_ab_C2.txt 2>&1; echo "C2 rc=$?"; cat gpurun_out/s3b_ab_C2.txt
timeout 600 python tools/ab.py --config C3 --reps 2 ab_libs/base.so ab_libs/xc.so > gpurun_out/s3b_ab_C3.txt 2>&1; echo "C3 rc=$?"; cat gpurun_out/s3b_ab_C3.txt
timeout 600 python tools/ab.py --config C1 --reps 3 --queries 4 ab_libs/base.so ab_libs/xc.so > gpurun_out/s3b_ab_C1.txt 2>&1; echo "C1 rc=$?"; cat gpurun_out/s3b_ab_C1.txt
