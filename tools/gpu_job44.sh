# Dev (GPU box): select size classes forked onto a side stream (A/B with UP_SELECT_FORK=0).
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_select.py tests/test_gpu_acceptance.py tests/test_gpu_golden_e2e.py tests/test_gpu_cascade.py tests/test_gpu_fullsize.py tests/test_gpu_meta.py -x -q > gpurun_out/pytest44.log 2>&1; echo "rc=$?" >> gpurun_out/pytest44.log
for F in 1 0; do
  echo "fork $F" >> gpurun_out/select44.txt; UP_SELECT_FORK=$F timeout 120 python tools/select_timing.py >> gpurun_out/select44.txt 2>&1
  UP_SELECT_FORK=$F timeout 400 python bench.py --skip-cpu --config c5 --e2e-steps 0 --steps 3 --warmup 3 > gpurun_out/bench44_c5_$F.log 2>&1
  UP_SELECT_FORK=$F timeout 400 python bench.py --skip-cpu --e2e-steps 0 --steps 5 --warmup 3 > gpurun_out/bench44_c2_$F.log 2>&1
done
