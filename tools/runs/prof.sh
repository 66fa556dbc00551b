#!/bin/bash
# tools/runs/prof.sh TAG LIB "CONFIG ARGS" ... : ncu --set full of the one-row K3 instance for each config
TAG=$1; LIB=$2; shift 2
mkdir -p gpurun_out
for cfg in "$@"; do
  tag=$(echo $cfg | cut -d' ' -f1)
  rep=/tmp/${TAG}_$tag
  KNNJOIN_LIB=$LIB timeout 900 python bench.py --config $cfg --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_plain_$tag.log 2>&1 || { echo "plain $tag failed"; continue; }
  KNNJOIN_LIB=$LIB timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
     -k "regex:${KREGEX:-k_accumulate_topk<\(int\)1, \(int\)\d, \(bool\)\d, \(int\)4, \(bool\)0, \(bool\)0>}" -s 1 -c 1 -f -o $rep \
     python bench.py --config $cfg --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_ncu_$tag.log 2>&1; echo "ncu $tag rc=$?"
  python tools/ncu_summary.py $rep.ncu-rep 30 > gpurun_out/${TAG}_${tag}_full.txt 2>&1
  python tools/ncu_lines.py $rep.ncu-rep 60 >> gpurun_out/${TAG}_${tag}_full.txt 2>&1
  python tools/ncu_peaks.py $rep.ncu-rep 40 > gpurun_out/${TAG}_${tag}_peaks.txt 2>&1
  python tools/ncu_lines.py $rep.ncu-rep 60 by-inst > gpurun_out/${TAG}_${tag}_byinst.txt 2>&1
  head -40 gpurun_out/${TAG}_${tag}_full.txt | grep -v "^  [A-Z]" 
done
