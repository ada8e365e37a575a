#!/usr/bin/env bash
# Dev sweep (GPU box): c1 (LLaMA 1x4K) scorer stage vs the scorer grid (UP_SCORE_GRID).
for G in ${GRIDS:-148 96 64 32 16}; do
  echo "GRID=$G $(UP_SCORE_GRID=$G SHAPE=llama4k timeout 120 python tools/score_timing.py) $(UP_SCORE_GRID=$G SHAPE=llama4k timeout 120 python tools/score_timing.py)"
done
