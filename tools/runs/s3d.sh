#!/bin/bash
# session 3, call d: windows inside one slice skip the entry lookup (fw) against HEAD (xc)
mkdir -p gpurun_out
V="ab_libs/xc.so ab_libs/fw.so"
timeout 900 python tools/ab.py --config C4 --rows-r 20000 --rows-s 2000000 --reps 2 $V > gpurun_out/s3d_ab_C4s.txt 2>&1; echo "C4s rc=$?"; cat gpurun_out/s3d_ab_C4s.txt
timeout 600 python tools/ab.py --config C2 --reps 3 --queries 4 $V > gpurun_out/s3d_ab_C2.txt 2>&1; echo "C2 rc=$?"; cat gpurun_out/s3d_ab_C2.txt
timeout 600 python tools/ab.py --config C3 --reps 2 $V > gpurun_out/s3d_ab_C3.txt 2>&1; echo "C3 rc=$?"; cat gpurun_out/s3d_ab_C3.txt
timeout 600 python tools/ab.py --config C5 --reps 2 $V > gpurun_out/s3d_ab_C5.txt 2>&1; echo "C5 rc=$?"; cat gpurun_out/s3d_ab_C5.txt
