#!/bin/bash
# slab plans (AMQFT_AB_SLAB=all) against the column / row / transpose four-step (none), v4
for dt in f32 f64; do
  for lg in 16 17 18 19 20 21 22 23 24 25 26; do
    if [ $dt = f64 ] && [ $lg -gt 24 ]; then continue; fi
    if [ $dt = f32 ] && [ $lg -lt 17 ]; then continue; fi
    tot=$([ $dt = f32 ] && echo 28 || echo 27)
    for m in all none; do
      echo -n "$m "; AMQFT_AB_SLAB=$m python tools/prof_fast.py --n $((1<<lg)) --batch $(( (1<<tot) >> lg )) --dtype $dt --iters 3
    done
  done
done
