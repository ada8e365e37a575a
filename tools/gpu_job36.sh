# Dev (GPU box): G=128 on score_tcw (HPC <= 2) + combine sid A/B.
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_scorer.py tests/test_gpu_golden_e2e.py tests/test_gpu_peer.py -q > gpurun_out/pytest36.log 2>&1; echo "rc=$?" >> gpurun_out/pytest36.log
for r in 1 2; do for s in llama gemma qwen; do echo "bcast $s $(SHAPE=$s timeout 120 python tools/score_timing.py 2>&1 | tail -1)" >> gpurun_out/score_timing36.txt; done; done
for s in gemma qwen mha; do echo "G128 $s $(G=128 SHAPE=$s timeout 120 python tools/score_timing.py 2>&1 | tail -1)" >> gpurun_out/score_timing36.txt; done
timeout 600 python bench.py --skip-cpu --e2e-steps 0 --config c4 --block-size 128 --steps 2 --warmup 1 > gpurun_out/bench36_c4_G128.log 2>&1
timeout 600 python bench.py --skip-cpu --e2e-steps 0 --config c3 --block-size 128 --steps 2 --warmup 1 > gpurun_out/bench36_c3_G128.log 2>&1
UP_NVCC_FLAGS="-DUP_COMBINE_SID_PER_HEAD" python paper_2605_06221_b200/build.py -f > /dev/null 2>&1
for r in 1 2; do for s in llama gemma qwen; do echo "perhead $s $(SHAPE=$s timeout 120 python tools/score_timing.py 2>&1 | tail -1)" >> gpurun_out/score_timing36.txt; done; done
python paper_2605_06221_b200/build.py -f > /dev/null 2>&1
