#!/usr/bin/env bash
# Dev sweep (GPU box): attention time vs UP_ATTN_POLY_PAIRS at the bench shapes.
set -u
mkdir -p gpurun_out
for P in ${PAIRS:-0 2 4 6}; do
  UP_NVCC_FLAGS="-DUP_ATTN_POLY_PAIRS=$P" python paper_2605_06221_b200/build.py -f > /dev/null
  echo "ATTN_POLY_PAIRS=$P"
  timeout 60 python tools/attn_probe.py 32768 32 8 128 0 | grep TFLOP
  timeout 60 python tools/attn_probe.py 8192,8192,8192,8192 32 8 128 0 | grep TFLOP
  timeout 60 python tools/attn_probe.py 32768 16 2 256 0 | grep TFLOP
done
python paper_2605_06221_b200/build.py -f > /dev/null
