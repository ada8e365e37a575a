#!/usr/bin/env bash
# Dev sweep (GPU box): two-tile attention vs ring depths and FMA-pipe exp2 pairs.
for V in "2 2 2" "3 2 2" "2 3 2" "2 2 3" "2 2 1"; do
  set -- $V
  UP_NVCC_FLAGS="-DUP_ATTN2_KST=$1 -DUP_ATTN2_VST=$2 -DUP_ATTN_POLY_PAIRS=$3" python paper_2605_06221_b200/build.py -f > /dev/null || { echo "build failed $V"; continue; }
  echo "KST=$1 VST=$2 NP=$3 $(timeout 60 python tools/attn_probe.py 32768 32 8 128 0 | grep TFLOP) $(timeout 60 python tools/attn_probe.py 8192,8192,8192,8192 32 8 128 0 | grep TFLOP)"
done
python paper_2605_06221_b200/build.py -f > /dev/null
