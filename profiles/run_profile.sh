#!/usr/bin/env bash
# Profiling recipe (run on the GPU box from the repo root, one GPU):
#   1. launch list with per-launch device time (cold-cache, serialised: compare SHARES)
#   2. one `ncu --set full` capture of each hot kernel (score_tcw_kernel, compact_copy_kernel,
#      select_radix_kernel, pair_weights_kernel, block_combine_kernel, expand_kernel,
#      scatter_rows_kernel = the reconstitution),
#      imported here with `ncu -i ... --page raw --csv` (profiles/summarize.py).
# CONFIG=c2 (default) or c3/c4; outputs go to $OUT (gpurun_out/ scratch); summaries are
# copied into profiles/ by summarize.py.
set -euo pipefail
OUT=${OUT:-gpurun_out}
CONFIG=${CONFIG:-c2}
TAG=${TAG:-}
mkdir -p "$OUT"
BENCH="python bench.py --config $CONFIG --steps 1 --warmup 1 --no-graph --e2e-steps 0 --skip-cpu --layer-sets 2"

ncu --metrics gpu__time_duration.sum --clock-control none -c 520 --csv \
    --log-file "$OUT/launches$TAG.csv" $BENCH > "$OUT/launches_bench$TAG.log" 2>&1 || true

ncu --set full --clock-control none --import-source on \
    -k regex:'score_tcw|compact_copy|select_radix|block_combine|pair_weights|expand_kernel|scatter_rows' -s 14 -c 7 \
    -o "$OUT/prof_full$TAG" -f $BENCH > "$OUT/prof_full$TAG.log" 2>&1 || true

# the drop layer's attention over the retained rows (bench.py attention stage, §8f row 1)
ncu --set full --clock-control none --import-source on -k regex:attention -c 1 \
    -o "$OUT/prof_attn$TAG" -f $BENCH > "$OUT/prof_attn$TAG.log" 2>&1 || true
