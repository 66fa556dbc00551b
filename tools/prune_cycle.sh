#!/bin/bash
# a6 pruned-query cycle: prune tests, the GPU suite, bench lines with and without pruning.  usage: TAG [alphas]
TAG=${1:-prune}; shift
ALPHAS=${*:-0.25 0.5 1.0}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_prune.py -q -x --timeout 600 > gpurun_out/${TAG}_prune_pytest.log 2>&1; echo "prune pytest rc=$?"; tail -15 gpurun_out/${TAG}_prune_pytest.log
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${TAG}_pytest.log
for c in C3 C5 C2; do
  for a in $ALPHAS; do
    timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --prune-alpha $a > gpurun_out/${TAG}_bench_${c}_a$a.json 2> gpurun_out/${TAG}_bench_${c}_a$a.err
    echo "bench $c alpha $a rc=$?"; python - <<PY
import json
j = json.load(open("gpurun_out/${TAG}_bench_${c}_a$a.json")); r = j["roofline"]; b = j["breakdown"]
print("${c} a=${a}", "step %.3f ms kernel %.3f ms" % (j["ms_per_step"], r["kernel_ms"]), b.get("counters"), {k: round(v, 3) for k, v in b["kernel_phase_share"].items()})
PY
  done
done
