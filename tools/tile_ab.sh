#!/bin/bash
# A/B runs of the in-shared-memory four-step (diagnostic build with
# AMQFT_TILE_AB in tile_v4.cu): AMQFT_TILE_KV = threads,CTAs/SM,prefetch
run() { echo -n "KV=$1 "; AMQFT_TILE_KV=$1 python tools/prof_fast.py --n $2 --batch $((268435456 / $2)) --iters 5; }
for kv in 64,4,0 64,4,1 64,5,1; do run $kv 4096; done
for kv in 64,4,0 64,4,1 64,6,1; do run $kv 2048; done
echo "swapped 64 x 32:"
for kv in 64,4,0 64,4,1 64,5,1; do AMQFT_TILE_SWAP=1 run $kv 2048; done
for kv in 64,0,0 64,0,1; do run $kv 512; done
AMQFT_TILE_SWAP=1 run 64,0,0 512
echo "defaults:"
for n in 256 512 1024 2048 4096; do python tools/prof_fast.py --n $n --batch $((268435456 / n)) --iters 5; done
