L=paper_1011_2807_b200/libknnjoin.so
for tpp in 1 2 62; do
timeout 900 ncu --metrics lts__t_sectors_srcunit_tex_lookup_hit.sum,lts__t_sectors_srcunit_tex_lookup_miss.sum,dram__bytes_read.sum,gpu__time_duration.sum,lts__t_requests_srcunit_tex.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum --clock-control none --kernel-name-base demangled -k 'regex:k_accumulate_topk<\(int\)1, \(int\)\d, \(bool\)\d, \(int\)4, \(bool\)0, \(bool\)0>' -s 1 -c 1 --csv --log-file gpurun_out/r3_l2_tpp$tpp.csv python tools/ab.py --config C5 --rows-r 4000 --reps 1 --queries 1 $L:tiles_per_pass=$tpp > /dev/null 2>&1
python3 - gpurun_out/r3_l2_tpp$tpp.csv $tpp <<'PY'
import sys,csv
rows=[r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
h=rows[0]
for r in rows[1:]:
    d=dict(zip(h,r)); print('tpp', sys.argv[2], d['Metric Name'], d['Metric Unit'], d['Metric Value'])
PY
done
