#!/usr/bin/env bash
# Dev sweep (GPU box): LLaMA scorer stage vs the FMA-pipe exp2 pairs (of 16) at D = 128.
for P in ${PAIRS:-3 4 5 6}; do
  UP_NVCC_FLAGS="-DUP_TCW_POLY_PAIRS_D128=$P" python paper_2605_06221_b200/build.py -f > /dev/null
  echo "NP=$P $(SHAPE=llama timeout 120 python tools/score_timing.py) $(SHAPE=llama timeout 120 python tools/score_timing.py)"
done
python paper_2605_06221_b200/build.py -f > /dev/null
