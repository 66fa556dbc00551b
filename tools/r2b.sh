set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import paper_1011_2807_b200" || exit 1
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/r2b_pytest.log 2>&1; echo pytest rc=$?
tail -30 gpurun_out/r2b_pytest.log
timeout 900 python bench.py > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err; echo bench rc=$?
head -c 2500 gpurun_out/r2b_bench.json; tail -5 gpurun_out/r2b_bench.err
