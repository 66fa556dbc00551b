#!/bin/bash
# quick timing of several configs (kernel/step ms, phase shares); usage: tools/quick.sh "C2 C3 C5" [extra bench args]
CS=$1; shift
for c in $CS; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline "$@" 2>/dev/null | python -c "
import json,sys; j=json.loads(sys.stdin.read()); r=j['roofline']; b=j['breakdown']
print('$c', 'step %.3f ms kernel %.3f ms frac %.3f' % (j['ms_per_step'], r['kernel_ms'], r['frac']), 'build %.2f' % b['build_index_ms'], {k: round(v, 3) for k, v in b['kernel_phase_share'].items()})"
done
