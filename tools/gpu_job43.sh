# Dev (GPU box): select size classes -- two launches (0) vs one 128x16 radix launch (1) vs one 512x4 radix launch (2).
set -u
mkdir -p gpurun_out
for P in 0 1 2; do
  UP_SELECT_PLAN=$P timeout 900 python -m pytest tests/test_gpu_select.py tests/test_gpu_acceptance.py tests/test_gpu_golden_e2e.py -x -q > gpurun_out/pytest43_$P.log 2>&1; echo "rc=$?" >> gpurun_out/pytest43_$P.log
  echo "plan $P" >> gpurun_out/select43.txt; UP_SELECT_PLAN=$P timeout 120 python tools/select_timing.py >> gpurun_out/select43.txt 2>&1
  UP_SELECT_PLAN=$P timeout 400 python bench.py --skip-cpu --config c5 --e2e-steps 0 --steps 3 --warmup 3 > gpurun_out/bench43_c5_$P.log 2>&1
done
