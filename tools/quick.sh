#!/bin/bash
# quick GPU check after a kernel change: core parity tests + one bench line per config (no e2e / cpu legs)
# usage: tools/quick.sh TAG [configs...]   (default configs: C2 C4 C3 C5)
TAG=${1:-q}; shift
CFGS=${@:-C2 C4 C3 C5}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 300 -p no:cacheprovider \
  -k "random_small or configs_scaled or head_feature or batch_sizes or multi_chunk or counters or row_order or split" \
  > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_pytest.log
for c in $CFGS; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
  python - "$c" "gpurun_out/${TAG}_bench_$c.json" <<'PY'
import json, sys
try:
    j = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    b = j["breakdown"]
    print(f"{sys.argv[1]}: step {j['ms_per_step']:.3f} ms  K3 {b['kernel_ms']:.3f} ms  build {b['build_index_ms']:.2f} ms  "
          f"frac {j['roofline']['frac']:.3f}  phases {b['kernel_phase_share']}  clocks {j['clocks'].get('sm_mhz')}")
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
done
