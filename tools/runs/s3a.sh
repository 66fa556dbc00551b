#!/bin/bash
# session 3, call a: scan microbenchmarks + A/B of the scan variants (exchange read+zero, theta every 4 steps, SHFL cum)
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mbscan tools/microbench_scan2.cu && timeout 120 /tmp/mbscan > gpurun_out/s3a_mbscan.txt 2>&1; echo "mb rc=$?"; cat gpurun_out/s3a_mbscan.txt
V="ab_libs/base.so ab_libs/xchg.so ab_libs/xth.so ab_libs/xts.so"
timeout 900 python tools/ab.py --config C4 --rows-r 20000 --rows-s 2000000 --reps 2 $V > gpurun_out/s3a_ab_C4s.txt 2>&1; echo "C4s rc=$?"; cat gpurun_out/s3a_ab_C4s.txt
timeout 600 python tools/ab.py --config C2 --reps 3 --queries 4 $V > gpurun_out/s3a_ab_C2.txt 2>&1; echo "C2 rc=$?"; cat gpurun_out/s3a_ab_C2.txt
timeout 600 python tools/ab.py --config C3 --reps 2 ab_libs/base.so ab_libs/xchg.so > gpurun_out/s3a_ab_C3.txt 2>&1; echo "C3 rc=$?"; cat gpurun_out/s3a_ab_C3.txt
timeout 600 python tools/ab.py --config C5 --reps 2 ab_libs/base.so ab_libs/xchg.so > gpurun_out/s3a_ab_C5.txt 2>&1; echo "C5 rc=$?"; cat gpurun_out/s3a_ab_C5.txt
