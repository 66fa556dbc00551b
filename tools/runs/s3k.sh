#!/bin/bash
# bench e2e with preallocated input slots: C2 / C1 lines (3 runs of C2) + the two-rank bench test
mkdir -p gpurun_out
for i in 1 2 3; do
timeout 300 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s3k_C2_$i.json 2> gpurun_out/s3k_C2_$i.err; echo "C2 rc=$?"
python -c "import json,sys; j=json.loads(open('gpurun_out/s3k_C2_$i.json').read().strip().splitlines()[-1]); print(j['ms_per_step'], j['e2e'])" 2>&1 | cut -c1-250
done
timeout 300 python bench.py --config C1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s3k_C1.json 2> gpurun_out/s3k_C1.err; echo "C1 rc=$?"
python -c "import json,sys; j=json.loads(open('gpurun_out/s3k_C1.json').read().strip().splitlines()[-1]); print(j['ms_per_step'], j['e2e'])" 2>&1 | cut -c1-250
timeout 600 python -m pytest tests/test_gpu_multirank.py -m gpu -q -x --timeout 500 -p no:cacheprovider 2>&1 | tail -2
