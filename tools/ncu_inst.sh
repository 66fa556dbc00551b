#!/bin/bash
# ncu --set full of the heads-path accumulate launch for C2 and a C4-shaped workload; per-line instruction counts
TAG=${1:-n}
for cfg in "C2" "C4 --rows-r 20000 --rows-s 2000000"; do
  tag=$(echo $cfg | cut -d' ' -f1)
  rep=/tmp/${TAG}_$tag
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_accumulate_topk -s 2 -c 1 -f -o $rep \
     python bench.py --config $cfg --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_ncu_$tag.log 2>&1; echo ncu $tag rc=$?
  python tools/ncu_summary.py $rep.ncu-rep 30 > gpurun_out/${TAG}_${tag}_full.txt 2>&1
  python tools/ncu_lines.py $rep.ncu-rep 60 >> gpurun_out/${TAG}_${tag}_full.txt 2>&1
  python tools/ncu_lines.py $rep.ncu-rep 150 by-inst > gpurun_out/${TAG}_${tag}_byinst.txt 2>&1
  head -12 gpurun_out/${TAG}_${tag}_full.txt | grep -E "Duration|Issue|instructions"
done
