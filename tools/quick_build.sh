#!/bin/bash
# Experiment helper: rebuild only the listed per-variant objects (e.g.
# "fast_v4") and relink, leaving the other objects as they are (stale code
# for the other variants: perf A/B of one variant only; run a full `make`
# before any test).
set -e
cd "$(dirname "$0")/../paper_1404_1810_b200/csrc"
for o in "$@"; do
  nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -Xptxas -v \
    --expt-relaxed-constexpr -c $o.cu -o build/$o.o 2> build/$o.o.ptxas.log || { cat build/$o.o.ptxas.log; exit 1; }
done
touch build/*.o
make -s
