#!/bin/bash
# final measurement cycle of session 3 (tools/round_cycle.sh r4b) + f4 streamed C4 at 8 / 32 / 64 blocks
bash tools/round_cycle.sh r4b
timeout 900 python tools/stream_bench.py --config C4 --blocks 8 32 64 --reps 2 > gpurun_out/r4b_stream_C4.jsonl 2> gpurun_out/r4b_stream_C4.err; echo "stream rc=$?"; cat gpurun_out/r4b_stream_C4.jsonl
