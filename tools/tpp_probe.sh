#!/bin/bash
# C5 pass-slab probe: kernel time and DRAM bytes of k_accumulate_topk vs tiles_per_pass.  usage: TAG CONFIG "tpps"
TAG=$1; C=$2; shift 2
mkdir -p gpurun_out
for t in $1; do
  timeout 300 python bench.py --config $C --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --tiles-per-pass $t > gpurun_out/${TAG}_${C}_tpp$t.json 2>/dev/null
  python -c "
import json; j=json.load(open('gpurun_out/${TAG}_${C}_tpp$t.json')); print('$C tpp=$t kernel %.2f ms step %.2f' % (j['roofline']['kernel_ms'], j['ms_per_step']))"
  timeout 300 ncu --metrics dram__bytes_read.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum --clock-control none -k regex:k_accumulate -s 3 -c 1 \
    python bench.py --config $C --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --tiles-per-pass $t 2>/dev/null | grep -E "dram__bytes|hit_rate|duration" | sed "s/^/  tpp=$t /"
done
