mkdir -p gpurun_out
for c in C3 C5; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_accumulate -s 1 -c 1 -o gpurun_out/r1c_${c}_prof \
      python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r1c_${c}_ncu.log 2>&1; echo "ncu $c rc=$?"
done
