#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/ab.py --config C4 --rows-r 20000 --rows-s 2000000 --reps 3 ab_libs/head4.so ab_libs/th2.so > gpurun_out/s3p_ab_C4s.txt 2>&1; echo "C4s rc=$?"; cat gpurun_out/s3p_ab_C4s.txt
timeout 240 python tools/ab.py --config C2 --reps 3 --queries 4 ab_libs/head4.so ab_libs/th2.so > gpurun_out/s3p_ab_C2.txt 2>&1; echo "C2 rc=$?"; cat gpurun_out/s3p_ab_C2.txt
