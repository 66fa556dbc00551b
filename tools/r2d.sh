timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/r2d_pytest.log 2>&1; echo pytest rc=$?
grep -E "passed|failed|FAILED" gpurun_out/r2d_pytest.log | head -40
for cfg in "C4 --rows-r 20000 --rows-s 2000000" "C5"; do
  tag=$(echo $cfg | cut -d' ' -f1)
  rep=/tmp/r2d_$tag
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_accumulate_topk -s 1 -c 1 -f -o $rep \
     python bench.py --config $cfg --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2d_ncu_$tag.log 2>&1; echo ncu $tag rc=$?
  python tools/ncu_summary.py $rep.ncu-rep 30 > gpurun_out/r2d_${tag}_full.txt 2>&1
  python tools/ncu_lines.py $rep.ncu-rep 80 >> gpurun_out/r2d_${tag}_full.txt 2>&1
  ncu -i $rep.ncu-rep --page source --csv > gpurun_out/r2d_${tag}_source.csv 2>/dev/null
done
