#!/bin/bash
# A/B of libknnjoin variants on C4s / C2 / C3 / C5 with short per-config timeouts: tools/runs/ab4s.sh TAG base.so variant.so ...
TAG=$1; shift
mkdir -p gpurun_out
V="$@"
timeout 300 python tools/ab.py --config C4 --rows-r 20000 --rows-s 2000000 --reps 2 $V > gpurun_out/${TAG}_ab_C4s.txt 2>&1; echo "C4s rc=$?"; cat gpurun_out/${TAG}_ab_C4s.txt
timeout 240 python tools/ab.py --config C2 --reps 3 --queries 4 $V > gpurun_out/${TAG}_ab_C2.txt 2>&1; echo "C2 rc=$?"; cat gpurun_out/${TAG}_ab_C2.txt
timeout 240 python tools/ab.py --config C3 --reps 2 $V > gpurun_out/${TAG}_ab_C3.txt 2>&1; echo "C3 rc=$?"; cat gpurun_out/${TAG}_ab_C3.txt
timeout 300 python tools/ab.py --config C5 --reps 2 $V > gpurun_out/${TAG}_ab_C5.txt 2>&1; echo "C5 rc=$?"; cat gpurun_out/${TAG}_ab_C5.txt
timeout 120 python tools/ab.py --config C1 --reps 3 --queries 4 $V > gpurun_out/${TAG}_ab_C1.txt 2>&1; echo "C1 rc=$?"; cat gpurun_out/${TAG}_ab_C1.txt
