#!/usr/bin/env bash
# Dev sweep (GPU box): bench value vs the PDL family mask (score 1, select 2, compact 4,
# meta 8, compaction scans 16), per config.
for C in ${CONFIGS:-c2}; do
for R in 1 2; do
for M in ${MASKS:-11 0}; do
  echo "$C MASK=$M $(UP_PDL_MASK=$M timeout 300 python bench.py --config $C --skip-cpu --e2e-steps 0 --steps 5 | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]/1e6,1), round(d["ms_per_step"],3))')"
done; done; done
