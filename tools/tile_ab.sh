#!/bin/bash
# A/B runs of the in-shared-memory four-step (diagnostic build with
# AMQFT_TILE_AB in tile_v4.cu): AMQFT_TILE_KV = instance key (tile_kernel.cuh make_tile)
export AMQFT_AB_TILE=16,65536
echo "2^15: cluster of 2, 32x32x32 T=512 | cluster of 4, T=256 x 2 CTAs"
AMQFT_TILE_KV=512,0,0 timeout 120 python tools/tile_check.py 4 15 2>&1 | head -1
AMQFT_TILE_KV=256,0,0 timeout 120 python tools/tile_check.py 4 15 2>&1 | head -1
echo "2^16: cluster of 4, 32x32x64 T=256 | cluster of 8 T=128 x2: 32x32x64 | 64x32x32"
AMQFT_TILE_KV=256,0,0 timeout 120 python tools/tile_check.py 4 16 2>&1 | head -1
AMQFT_TILE_KV=128,0,0 timeout 120 python tools/tile_check.py 4 16 2>&1 | head -1
AMQFT_TILE_KV=129,0,0 timeout 120 python tools/tile_check.py 4 16 2>&1 | head -1
