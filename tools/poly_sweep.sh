#!/usr/bin/env bash
# Dev sweep (GPU box): exp2 throughput probe + scorer time vs UP_POLY_PAIRS.
set -u
mkdir -p gpurun_out tools/_bin
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -o tools/_bin/ubench_ex2 tools/ubench_ex2.cu && tools/_bin/ubench_ex2
for P in ${PAIRS:-0 2 4 6 8}; do
  UP_NVCC_FLAGS="-DUP_POLY_PAIRS=$P" python paper_2605_06221_b200/build.py -f > /dev/null
  echo "POLY_PAIRS=$P"; REGIME=planted python tools/score_timing.py; REGIME=iid python tools/score_timing.py
done
python paper_2605_06221_b200/build.py -f > /dev/null
