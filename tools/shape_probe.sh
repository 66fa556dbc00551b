#!/bin/bash
# kernel time vs (tile, batch_rows, cta_warps).  usage: TAG "C5:8192:0:0 C5:16384:1:4 ..."
TAG=$1; shift
mkdir -p gpurun_out
for s in $1; do
  IFS=: read c t b w <<< "$s"
  timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --tile $t --batch-rows $b --cta-warps $w > gpurun_out/${TAG}_$c_$t_$b_$w.json 2>/dev/null
  python -c "
import json; j=json.load(open('gpurun_out/${TAG}_$c_$t_$b_$w.json')); b=j['breakdown']
print('$s kernel %.2f ms step %.2f' % (j['roofline']['kernel_ms'], j['ms_per_step']), {k: round(v, 3) for k, v in b['kernel_phase_share'].items()})" 2>/dev/null || echo "$s failed"
done
