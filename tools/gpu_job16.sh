# Dev (GPU box): ablation-shape envelope (G, n), pair_weights merge, C++ engine loop.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scorer.py tests/test_gpu_golden_e2e.py tests/test_gpu_peer.py -q > gpurun_out/pytest16.log 2>&1; echo "rc=$?" >> gpurun_out/pytest16.log
timeout 300 python bench.py --skip-cpu --config c3-rank --e2e-steps 0 > gpurun_out/bench16_c3rank.log 2>&1
for G in 32 128; do timeout 300 python bench.py --skip-cpu --e2e-steps 0 --block-size $G > gpurun_out/bench16_c2_G$G.log 2>&1; done
timeout 300 python bench.py --skip-cpu --e2e-steps 0 --query-window 32 > gpurun_out/bench16_c2_n32.log 2>&1
timeout 900 python bench.py --skip-cpu --e2e-steps 0 --query-window 512 --steps 2 --warmup 1 --layer-sets 2 > gpurun_out/bench16_c2_n512.log 2>&1
timeout 300 examples/_build/drop_layer_bench > gpurun_out/cpp16.log 2>&1
