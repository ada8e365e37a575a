# Dev (GPU box): parity epilogues walk only their own subtiles.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scorer.py tests/test_gpu_golden_e2e.py tests/test_gpu_peer.py -x -q > gpurun_out/pytest57.log 2>&1; echo "rc=$?" >> gpurun_out/pytest57.log
for r in 1 2; do for s in mha mha256 gqa2 gemma qwen llama; do echo "$s $(SHAPE=$s timeout 120 python tools/score_timing.py 2>&1 | tail -1)" >> gpurun_out/score_timing57.txt; done; done
for s in mha gqa2; do echo "G128 $s $(G=128 SHAPE=$s timeout 120 python tools/score_timing.py 2>&1 | tail -1)" >> gpurun_out/score_timing57.txt; done
