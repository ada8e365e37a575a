# Dev (GPU box): CTA-counter parity in score_tcw (HPC 2/1) + G=128 on D<=128 + e2e double buffering.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scorer.py -x -q > gpurun_out/pytest37.log 2>&1; echo "rc=$?" >> gpurun_out/pytest37.log
timeout 600 python -m pytest tests/test_gpu_golden_e2e.py tests/test_gpu_peer.py tests/test_gpu_cascade.py -x -q > gpurun_out/pytest37b.log 2>&1; echo "rc=$?" >> gpurun_out/pytest37b.log
for s in llama gemma qwen mha mha256 gqa2 mixed; do echo "G64 $s $(SHAPE=$s timeout 120 python tools/score_timing.py 2>&1 | tail -1)" >> gpurun_out/score_timing37.txt; done
for s in mha gqa2; do echo "G128 $s $(G=128 SHAPE=$s timeout 120 python tools/score_timing.py 2>&1 | tail -1)" >> gpurun_out/score_timing37.txt; done
timeout 600 python bench.py --skip-cpu --steps 3 --warmup 3 > gpurun_out/bench37_c2.log 2>&1
