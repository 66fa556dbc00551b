#!/bin/bash
# full measurement cycle on the GPU box: parity tests, the default bench line, the launch list and one
# ncu --set full capture of the accumulate kernel (each ncu pass only after the same command exited 0 without
# ncu; the .ncu-rep stays in /tmp on the box and is summarised to text here, since gpurun returns <= 64 MiB),
# plus one bench line per other config.   usage: tools/round_cycle.sh TAG [configs...]
TAG=${1:-run}; shift
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > gpurun_out/${TAG}_smi.txt
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${TAG}_pytest.log
timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"; head -c 1500 gpurun_out/${TAG}_bench.json; echo
if timeout 300 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_plain.log 2>&1; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv \
      python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
  rep=/tmp/${TAG}_prof
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_accumulate -s 2 -c 1 -f -o $rep \
      python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu full rc=$?"
  python tools/ncu_summary.py $rep.ncu-rep 30 > gpurun_out/${TAG}_C2_full.txt 2>&1
  python tools/ncu_lines.py $rep.ncu-rep 40 >> gpurun_out/${TAG}_C2_full.txt 2>&1
  ncu -i $rep.ncu-rep --page raw --csv > gpurun_out/${TAG}_C2_raw.csv 2>/dev/null
fi
for c in "$@"; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
  echo "bench $c rc=$?"; head -c 600 gpurun_out/${TAG}_bench_$c.json; echo
done
