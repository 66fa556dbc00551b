timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_precision.py -m gpu -q -x --timeout 600 -p no:cacheprovider -k "head or multi_chunk or layout or dynamic" 2>&1 | tail -2
timeout 900 python tools/head_phases.py C4 20000 2000000 "32:0.125" "40:0.0625" "48:0.03125" "64:0.03125" 2>&1 | tail -4
