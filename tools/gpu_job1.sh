set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
for s in llama llama4k gemma qwen qwen-tp8; do
  echo "tcw $(SHAPE=$s timeout 120 python tools/score_timing.py 2>&1 | tail -1)" >> gpurun_out/score_timing.txt
  echo "tc2 $(UP_TC2=1 SHAPE=$s timeout 120 python tools/score_timing.py 2>&1 | tail -1)" >> gpurun_out/score_timing.txt
done
timeout 400 python bench.py > gpurun_out/bench_c2.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1
