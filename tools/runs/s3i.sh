#!/bin/bash
# session 3, call i: predicated per-row atomics (fixed: no early return before the vote) and ld2, short timeouts
mkdir -p gpurun_out
for V in ab_libs/pred.so ab_libs/ld2.so; do
  timeout 240 python tools/ab.py --config C2 --reps 3 --queries 4 ab_libs/head1.so $V > gpurun_out/s3i_ab_C2_$(basename $V .so).txt 2>&1; echo "C2 $V rc=$?"; cat gpurun_out/s3i_ab_C2_$(basename $V .so).txt
  timeout 300 python tools/ab.py --config C4 --rows-r 20000 --rows-s 2000000 --reps 2 ab_libs/head1.so $V > gpurun_out/s3i_ab_C4s_$(basename $V .so).txt 2>&1; echo "C4s $V rc=$?"; cat gpurun_out/s3i_ab_C4s_$(basename $V .so).txt
done
