#!/bin/bash
# round-end evidence on the final code: microbenchmarks (smem atomics / L2 / HBM peaks the roofline needs), smoke,
# then tools/round_cycle.sh (GPU tests, bench lines, launch list, ncu C2).  usage: TAG
TAG=$1
mkdir -p gpurun_out
timeout 300 ./tools/microbench > gpurun_out/${TAG}_microbench.txt 2>&1; echo "microbench rc=$?"; tail -12 gpurun_out/${TAG}_microbench.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
bash tools/round_cycle.sh $TAG C1 C3 C4 C5
