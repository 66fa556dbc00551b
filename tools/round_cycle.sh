#!/bin/bash
# Full measurement cycle on the GPU box (tools/round_cycle.sh TAG): GPU tests, smoke, the driver's default bench line
# (C4), one line per other config, the launch list of the bench command, ncu DRAM traffic of K3 on full C4 and
# ncu --set full captures (C4-shaped, C2, C3, C5).  Every ncu pass runs only after the same command exited 0 without
# ncu; summaries go to gpurun_out/ (profiles/ keeps the committed copies).
TAG=${1:-run}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > gpurun_out/${TAG}_smi.txt
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${TAG}_smoke.log
timeout 1200 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"; head -c 800 gpurun_out/${TAG}_bench.json; echo
for c in C2 C1 C3 C5; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
  echo "bench $c rc=$?"
done
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
if timeout 900 $B > gpurun_out/${TAG}_plain.log 2>&1; then
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv \
     $B > gpurun_out/${TAG}_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
  timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,gpu__time_duration.sum --clock-control none \
     --kernel-name-base demangled -k "regex:k_accumulate_topk<\(int\)2, \(int\)\d, \(bool\)\d, \(int\)8, \(bool\)1, \(bool\)0>" -s 1 -c 1 --csv --log-file gpurun_out/${TAG}_C4_dram.csv $B > gpurun_out/${TAG}_ncu_dram.log 2>&1; echo "ncu dram rc=$?"
fi
# ncu --set full of the K3 instance each config runs (the gated-out candidate shape returns at entry and is skipped)
HEADS='k_accumulate_topk<\(int\)2, \(int\)\d, \(bool\)\d, \(int\)8, \(bool\)1, \(bool\)0>'
ROWP='k_accumulate_topk<\(int\)1, \(int\)\d, \(bool\)\d, \(int\)4, \(bool\)0, \(bool\)0>'
for cfg in "C4 --rows-r 20000 --rows-s 2000000" "C2" "C3" "C5"; do
  tag=$(echo $cfg | cut -d' ' -f1); [ "$cfg" != "C4" ] && [ "$tag" = "C4" ] && tag=C4s
  case $tag in C3|C5) KR=$ROWP ;; *) KR=$HEADS ;; esac
  rep=/tmp/${TAG}_$tag
  timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$KR" -s 1 -c 1 -f -o $rep \
     python bench.py --config $cfg --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_ncu_$tag.log 2>&1; echo "ncu full $tag rc=$?"
  python tools/ncu_summary.py $rep.ncu-rep 30 > gpurun_out/${TAG}_${tag}_full.txt 2>&1
  python tools/ncu_lines.py $rep.ncu-rep 60 >> gpurun_out/${TAG}_${tag}_full.txt 2>&1
  python tools/ncu_peaks.py $rep.ncu-rep 40 > gpurun_out/${TAG}_${tag}_peaks.txt 2>&1
  python tools/ncu_lines.py $rep.ncu-rep 100 by-inst > gpurun_out/${TAG}_${tag}_byinst.txt 2>&1
done
