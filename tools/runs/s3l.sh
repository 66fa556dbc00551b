#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/ab.py --config C5 --reps 2 ab_libs/head2.so ab_libs/vf.so > gpurun_out/s3l_ab_C5.txt 2>&1; echo "C5 rc=$?"; cat gpurun_out/s3l_ab_C5.txt
