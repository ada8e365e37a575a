# Dev (GPU box): fused scorer tail for small launches.
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_scorer.py tests/test_gpu_golden_e2e.py tests/test_gpu_cascade.py tests/test_gpu_peer.py tests/test_gpu_select.py tests/test_gpu_compact.py -q > gpurun_out/pytest20.log 2>&1; echo "rc=$?" >> gpurun_out/pytest20.log
for s in llama4k llama; do
  echo "auto $(SHAPE=$s timeout 120 python tools/score_timing.py 2>&1 | tail -1)" >> gpurun_out/score_timing20.txt
  echo "nofuse $(UP_FUSED_TAIL=0 SHAPE=$s timeout 120 python tools/score_timing.py 2>&1 | tail -1)" >> gpurun_out/score_timing20.txt
done
echo "fuse-forced $(UP_FUSED_TAIL=1 SHAPE=llama timeout 120 python tools/score_timing.py 2>&1 | tail -1)" >> gpurun_out/score_timing20.txt
timeout 300 python bench.py --skip-cpu --config c1 --e2e-steps 0 > gpurun_out/bench20_c1.log 2>&1
UP_FUSED_TAIL=0 timeout 300 python bench.py --skip-cpu --config c1 --e2e-steps 0 > gpurun_out/bench20_c1_nofuse.log 2>&1
timeout 300 python bench.py --skip-cpu --e2e-steps 0 > gpurun_out/bench20_c2.log 2>&1
