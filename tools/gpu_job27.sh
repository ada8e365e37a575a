# Dev (GPU box): HPC=1 parity fix -- parity + timings.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_scorer.py tests/test_gpu_golden_e2e.py tests/test_gpu_peer.py tests/test_gpu_acceptance.py tests/test_gpu_cascade.py -q > gpurun_out/pytest27.log 2>&1; echo "rc=$?" >> gpurun_out/pytest27.log
for s in mha mha256 llama; do echo "tcw1 $(SHAPE=$s timeout 120 python tools/score_timing.py 2>&1 | tail -1)" >> gpurun_out/score_timing27.txt; done
timeout 600 python bench.py --skip-cpu --e2e-steps 0 --query-window 32 > gpurun_out/bench27_c2_n32.log 2>&1
timeout 600 python bench.py --skip-cpu --e2e-steps 0 --query-window 64 > gpurun_out/bench27_c2_n64.log 2>&1
