#!/bin/bash
# one build->measure cycle on the GPU box: parity tests, a bench line, and an ncu --set full capture of the
# accumulate kernel (only after the same bench command exited 0 without ncu).
# usage: tools/gpu_cycle.sh TAG [bench args...]
TAG=${1:-run}; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${TAG}_pytest.log
python bench.py "$@" > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"; cat gpurun_out/${TAG}_bench.json | head -c 3000; echo
python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline "$@" > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_accumulate -s 2 -c 1 -o gpurun_out/${TAG}_prof \
    python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline "$@" > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu rc=$?"
