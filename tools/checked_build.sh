#!/bin/bash
# Checked build (T9 without compute-sanitizer, which this pool does not allow): the library with -DKJ_CHECKS
# (device-side bounds checks on every shared / global index the kernels form; a failure prints its site and traps)
# -> ab_libs/checked/libknnjoin.so.  Run anything against it with KNNJOIN_LIB=ab_libs/checked/libknnjoin.so.
set -e
mkdir -p ab_libs/checked
KJ_EXTRA_NVCC_FLAGS="-DKJ_CHECKS" python paper_1011_2807_b200/build.py --src paper_1011_2807_b200/csrc --out $(pwd)/ab_libs/checked/libknnjoin.so
