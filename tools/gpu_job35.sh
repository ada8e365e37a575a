# Dev (GPU box): combine sid broadcast; G=128 / n=32 envelope rows for Gemma & Qwen.
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_scorer.py tests/test_gpu_golden_e2e.py tests/test_gpu_peer.py tests/test_gpu_acceptance.py -q > gpurun_out/pytest35.log 2>&1; echo "rc=$?" >> gpurun_out/pytest35.log
for s in llama llama4k gemma qwen qwen-tp8; do echo "$s $(SHAPE=$s timeout 120 python tools/score_timing.py 2>&1 | tail -1)" >> gpurun_out/score_timing35.txt; done
timeout 600 python bench.py --skip-cpu --e2e-steps 0 > gpurun_out/bench35_c2.log 2>&1
timeout 600 python bench.py --skip-cpu --e2e-steps 0 --config c4 --block-size 128 --steps 2 --warmup 1 > gpurun_out/bench35_c4_G128.log 2>&1
timeout 600 python bench.py --skip-cpu --e2e-steps 0 --config c4 --query-window 32 --steps 2 --warmup 1 > gpurun_out/bench35_c4_n32.log 2>&1
timeout 600 python bench.py --skip-cpu --e2e-steps 0 --config c3 --block-size 128 --steps 2 --warmup 1 > gpurun_out/bench35_c3_G128.log 2>&1
