#!/bin/bash
# fp32 CDFT throughput per size on one GPU (diagnostic): 2^28 reals per launch
# (1 GiB in), variant 4, fast order -> the path the plan picks per N.
for lg in $(seq 1 20); do
  n=$((1 << lg))
  python tools/prof_fast.py --n $n --batch $((268435456 / n)) --dtype f32
done
