#!/bin/bash
# Config 2's twiddles w_N^(n2 k1): read from the host-built table (coalesced __ldg, the default) or
# computed on the fly (sincospif of the exact integer phase) -- the north-star's choice "by measured
# GB/s".  Output committed as profiles/r02_tile_twiddle_ab.log.
echo "table:"
python tools/prof_fast.py --n 4096 --batch 65536 --iters 10
python tools/check_v.py 4 4096
echo "on the fly (AMQFT_AB_TILE_TW=fly):"
AMQFT_AB_TILE_TW=fly python tools/prof_fast.py --n 4096 --batch 65536 --iters 10
AMQFT_AB_TILE_TW=fly python tools/check_v.py 4 4096
