#!/bin/bash
# quick parameter sweep of bench.py (kernel/step ms only); usage: tools/sweep.sh TAG "args1" "args2" ...
TAG=$1; shift
for a in "$@"; do
  echo "== $a"
  python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline $a 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('value %.4e step %.3f ms kernel %.3f ms frac %.3f' % (j['value'], j['ms_per_step'], j['roofline']['kernel_ms'], j['roofline']['frac']), j['breakdown'].get('kernel_phase_share'), 'build %.3f prep %.3f' % (j['breakdown']['build_index_ms'], j['breakdown']['query_prep_ms']), j['breakdown']['counters'])"
done 2>&1 | tee gpurun_out/${TAG}_sweep.txt
