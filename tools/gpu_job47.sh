# Dev (GPU box): pair_weights templated on CTA size (32-warp CTA path restored for spread pairs).
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scorer.py tests/test_gpu_peer.py tests/test_gpu_golden_e2e.py -x -q > gpurun_out/pytest47.log 2>&1; echo "rc=$?" >> gpurun_out/pytest47.log
for s in llama4k mixed-llama qwen-tp8; do echo "$s $(SHAPE=$s timeout 120 python tools/score_timing.py 2>&1 | tail -1)" >> gpurun_out/score_timing47.txt; done
timeout 300 python bench.py --skip-cpu --config c3-rank --e2e-steps 0 --steps 3 --warmup 3 > gpurun_out/bench47_c3rank.log 2>&1
timeout 300 python bench.py --skip-cpu --config c1 --e2e-steps 0 --steps 20 --warmup 5 > gpurun_out/bench47_c1.log 2>&1
