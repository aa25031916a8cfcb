#!/bin/bash
# Round profiling recipe (run on the GPU box from the repo root):
#   1. the bench line (no profiler)                 -> gpurun_out/bench_n1.json
#   2. the launch list of a short bench run (ncu)   -> gpurun_out/launches.csv
#   3. one --set full capture of the top kernel     -> gpurun_out/k_top_full.ncu-rep
#      (config 2: k_tile, the in-shared-memory four-step; AMQFT_AB_TILE=none: k_fast)
# Each ncu pass runs only after the same command exited 0 without ncu.
set -u
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_n1.log 2>&1 || { tail -5 gpurun_out/bench_n1.log; exit 1; }
tail -1 gpurun_out/bench_n1.log > gpurun_out/bench_n1.json
SHORT="python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-all-variants"
$SHORT > gpurun_out/short.log 2>&1 || { tail -5 gpurun_out/short.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $SHORT \
  > gpurun_out/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k 'regex:k_tile|k_fast' -s 3 -c 1 \
  -o gpurun_out/k_top_full -f $SHORT > gpurun_out/ncu_full.log 2>&1
echo "profile_round: done"
