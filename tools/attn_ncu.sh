#!/usr/bin/env bash
# Dev (GPU box): one ncu --set full capture of the attention kernel at the LLaMA 32K shape.
mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:attention -s 1 -c 1 \
  -o gpurun_out/prof_attn -f python tools/attn_probe.py 32768 32 8 128 0 > gpurun_out/prof_attn.log 2>&1
