#!/bin/bash
# tools/ncu_one.sh TAG KERNEL_REGEX SKIP "bench args": ncu --set full of one launch + per-line summaries
TAG=$1; KR=$2; SKIP=$3; shift 3
rep=/tmp/${TAG}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KR -s $SKIP -c 1 -f -o $rep \
   python bench.py $@ --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_ncu.log 2>&1; echo ncu rc=$?
python tools/ncu_summary.py $rep.ncu-rep 30 > gpurun_out/${TAG}_full.txt 2>&1
python tools/ncu_lines.py $rep.ncu-rep 60 >> gpurun_out/${TAG}_full.txt 2>&1
python tools/ncu_lines.py $rep.ncu-rep 150 by-inst > gpurun_out/${TAG}_byinst.txt 2>&1
head -45 gpurun_out/${TAG}_full.txt
