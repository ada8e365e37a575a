# Dev (GPU box): score_tcw HPC=1 (MHA, full row packing) A/B + parity.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_scorer.py tests/test_gpu_golden_e2e.py tests/test_gpu_peer.py tests/test_gpu_acceptance.py -q > gpurun_out/pytest26.log 2>&1; echo "rc=$?" >> gpurun_out/pytest26.log
for s in mha mha256 llama; do echo "tcw1 $(SHAPE=$s timeout 120 python tools/score_timing.py 2>&1 | tail -1)" >> gpurun_out/score_timing26.txt; done
timeout 600 python bench.py --skip-cpu --e2e-steps 0 --query-window 32 > gpurun_out/bench26_c2_n32.log 2>&1
UP_NVCC_FLAGS="-DUP_NO_TCW_HPC1" python paper_2605_06221_b200/build.py -f > /dev/null 2>&1
for s in mha mha256; do echo "tc1 $(SHAPE=$s timeout 120 python tools/score_timing.py 2>&1 | tail -1)" >> gpurun_out/score_timing26.txt; done
python paper_2605_06221_b200/build.py -f > /dev/null 2>&1
