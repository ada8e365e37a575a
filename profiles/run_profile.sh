#!/usr/bin/env bash
# Profiling recipe (run on the GPU box from the repo root, one GPU):
#   1. launch list with per-launch device time (cold-cache, serialised: compare SHARES)
#   2. one `ncu --set full` capture of each hot kernel (score_tc4_kernel, compact_copy_kernel,
#      select_radix_kernel, block_combine_kernel, expand_kernel), imported here with `ncu -i ... --page raw --csv`.
# Outputs go to gpurun_out/ (scratch); summaries are copied into profiles/ by hand.
set -euo pipefail
OUT=${OUT:-gpurun_out}
mkdir -p "$OUT"
BENCH="python bench.py --config c2 --steps 1 --warmup 1 --no-graph --e2e-steps 0 --skip-cpu --layer-sets 2"

ncu --metrics gpu__time_duration.sum --clock-control none -c 520 --csv \
    --log-file "$OUT/launches.csv" $BENCH > "$OUT/launches_bench.log" 2>&1 || true

ncu --set full --clock-control none --import-source on \
    -k regex:'score_tcw|compact_copy|select_radix|block_combine|pair_weights|expand_kernel' -s 12 -c 6 \
    -o "$OUT/prof_full" -f $BENCH > "$OUT/prof_full.log" 2>&1 || true
