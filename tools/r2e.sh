nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mbcopy tools/microbench_copy.cu && timeout 300 /tmp/mbcopy > gpurun_out/r2e_mbcopy.txt 2>&1; echo mb rc=$?
cat gpurun_out/r2e_mbcopy.txt
rep=/tmp/r2e_C4
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_accumulate_topk -s 2 -c 1 -f -o $rep \
   python bench.py --config C4 --rows-r 20000 --rows-s 2000000 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2e_ncu_C4.log 2>&1; echo ncu rc=$?
python tools/ncu_summary.py $rep.ncu-rep 30 > gpurun_out/r2e_C4_full.txt 2>&1
python tools/ncu_lines.py $rep.ncu-rep 60 >> gpurun_out/r2e_C4_full.txt 2>&1
python tools/ncu_lines.py $rep.ncu-rep 120 by-inst > gpurun_out/r2e_C4_byinst.txt 2>&1
head -20 gpurun_out/r2e_C4_full.txt
