# Dev (GPU box): MMA warp issues heads out of order (A/B UP_TCW_OOO_MMA).
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scorer.py tests/test_gpu_golden_e2e.py tests/test_gpu_peer.py -x -q > gpurun_out/pytest58.log 2>&1; echo "rc=$?" >> gpurun_out/pytest58.log
for r in 1 2; do for s in llama llama4k gemma qwen mha gqa2; do echo "ooo $s $(SHAPE=$s timeout 120 python tools/score_timing.py 2>&1 | tail -1)" >> gpurun_out/score_timing58.txt; done; done
UP_NVCC_FLAGS="-DUP_TCW_OOO_MMA=0" python paper_2605_06221_b200/build.py -f > /dev/null 2>&1
for r in 1 2; do for s in llama llama4k gemma qwen mha gqa2; do echo "inorder $s $(SHAPE=$s timeout 120 python tools/score_timing.py 2>&1 | tail -1)" >> gpurun_out/score_timing58.txt; done; done
python paper_2605_06221_b200/build.py -f > /dev/null 2>&1
