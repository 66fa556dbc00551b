#!/bin/bash
# quick a6 check: prune tests, then bounded bench lines.  usage: TAG "C3:0.25 C3:0.1 ..."
TAG=$1; shift
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_prune.py -q -x --timeout 300 -m "gpu and not slow" > gpurun_out/${TAG}_prune_pytest.log 2>&1; echo "prune pytest rc=$?"; tail -15 gpurun_out/${TAG}_prune_pytest.log
for ca in $1; do
  c=${ca%%:*}; a=${ca##*:}
  timeout 240 python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --prune-alpha $a > gpurun_out/${TAG}_bench_${c}_a$a.json 2> gpurun_out/${TAG}_bench_${c}_a$a.err
  echo "bench $c alpha $a rc=$?"; python -c "
import json
j = json.load(open('gpurun_out/${TAG}_bench_${c}_a$a.json')); r = j['roofline']; b = j['breakdown']
print('${c} a=${a}', 'step %.3f ms kernel %.3f ms' % (j['ms_per_step'], r['kernel_ms']), b.get('counters'), {k: round(v, 3) for k, v in b['kernel_phase_share'].items()})" 2>/dev/null
done
