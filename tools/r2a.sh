set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import paper_1011_2807_b200" || python __graft_entry__.py build
timeout 600 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2a_bench_C4.json 2> gpurun_out/r2a_bench_C4.err; echo rc=$?
head -c 3000 gpurun_out/r2a_bench_C4.json
rep=/tmp/r2a_C4
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_accumulate -s 0 -c 1 -f -o $rep \
   python bench.py --config C4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2a_ncu.log 2>&1; echo ncu rc=$?
python tools/ncu_summary.py $rep.ncu-rep 30 > gpurun_out/r2a_C4_full.txt 2>&1
python tools/ncu_lines.py $rep.ncu-rep 60 >> gpurun_out/r2a_C4_full.txt 2>&1
ncu -i $rep.ncu-rep --page raw --csv > gpurun_out/r2a_C4_raw.csv 2>/dev/null
ncu -i $rep.ncu-rep --page source --csv > gpurun_out/r2a_C4_source.csv 2>/dev/null
ls -la gpurun_out | tail
