#!/bin/bash
# session 3, call h: A/B of two windows in flight on the block path (ld2) and predicated per-row atomics (pred);
# f4 streamed C4 against resident
mkdir -p gpurun_out
bash tools/runs/ab4.sh s3h ab_libs/head1.so ab_libs/ld2.so ab_libs/pred.so
timeout 900 python tools/stream_bench.py --config C4 --blocks 8 16 --reps 2 > gpurun_out/s3h_stream_C4.jsonl 2> gpurun_out/s3h_stream_C4.err; echo "stream rc=$?"; cat gpurun_out/s3h_stream_C4.jsonl; tail -3 gpurun_out/s3h_stream_C4.err
