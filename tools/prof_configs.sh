#!/bin/bash
# ncu --set full of the accumulate kernel for each config given; summarised to text on the box (the .ncu-rep
# files are ~36 MB each and would exceed gpurun's 64 MiB return limit).  usage: tools/prof_configs.sh TAG C3 C5 ...
TAG=$1; shift
mkdir -p gpurun_out
for c in "$@"; do
  rep=/tmp/${TAG}_${c}_prof
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_accumulate -s 1 -c 1 -f -o $rep \
      python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_${c}_ncu.log 2>&1
  echo "ncu $c rc=$?"
  python tools/ncu_summary.py $rep.ncu-rep 30 > gpurun_out/${TAG}_${c}_full.txt 2>&1
  python tools/ncu_lines.py $rep.ncu-rep 40 >> gpurun_out/${TAG}_${c}_full.txt 2>&1
  ncu -i $rep.ncu-rep --page raw --csv > gpurun_out/${TAG}_${c}_raw.csv 2>/dev/null
done
