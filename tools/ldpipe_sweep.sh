#!/usr/bin/env bash
# Dev sweep (GPU box): scorer stage time with / without the pipelined TMEM loads.
for P in 0 1; do
  UP_NVCC_FLAGS="-DUP_TCW_LD_PIPE=$P" python paper_2605_06221_b200/build.py -f > /dev/null
  echo "LD_PIPE=$P"
  for S in llama gemma qwen-tp8; do SHAPE=$S timeout 120 python tools/score_timing.py; SHAPE=$S timeout 120 python tools/score_timing.py; done
done
python paper_2605_06221_b200/build.py -f > /dev/null
