#!/bin/bash
# A/B runs of the in-shared-memory four-step (diagnostic build with
# AMQFT_TILE_AB in tile_v4.cu): AMQFT_TILE_KV = instance key (tile_kernel.cuh make_tile)
run() { echo -n "KV=$1 "; AMQFT_TILE_KV=$1 python tools/prof_fast.py --n $2 --batch $((268435456 / $2)) --iters 5; }
echo "8192: 16x16x32 T=256x2 | 32x16x16 T=256x2 | 16x32x16 T=256x2 | 32x16x16 T=512"
for k in 256 257 258 512; do run $k,0,0 8192; done
echo "16384: 32x16x32 T=512 | 32x32x16 T=512 | 32x16x32 T=256"
for k in 513 514 515; do run $k,0,0 16384; done
echo "8: 2x4 | 4x2 | direct"
export AMQFT_AB_TILE=8,16384
for k in 64 65; do run $k,0,0 8; done
AMQFT_AB_TILE=none python tools/prof_fast.py --n 8 --batch 33554432 --iters 5
