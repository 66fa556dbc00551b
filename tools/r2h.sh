for hm in 16 24 32; do
  python bench.py --config C4 --steps 2 --warmup 2 --no-e2e --no-cpu-baseline --head-max $hm > gpurun_out/r2h_$hm.json 2>/dev/null
  python -c "
import json; j=json.loads(open('gpurun_out/r2h_$hm.json').read().strip().splitlines()[-1]); b=j['breakdown']
print('head_max $hm', 'K3', round(b['kernel_ms'],1), 'phases', b['kernel_phase_share'], 'counters', b['counters'])"
done
