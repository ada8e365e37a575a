# Dev (GPU box): lean path for the parity epilogues (HPC 2 / 1, G = 64), A/B.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scorer.py tests/test_gpu_golden_e2e.py tests/test_gpu_peer.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest50.log 2>&1; echo "rc=$?" >> gpurun_out/pytest50.log
for r in 1 2; do for s in gemma qwen qwen-tp8 mha gqa2 mha256; do echo "lean2 $s $(SHAPE=$s timeout 120 python tools/score_timing.py 2>&1 | tail -1)" >> gpurun_out/score_timing50.txt; done; done
timeout 400 python bench.py --skip-cpu --config c4 --e2e-steps 0 --steps 3 --warmup 3 > gpurun_out/bench50_c4.log 2>&1
timeout 400 python bench.py --skip-cpu --config c3 --e2e-steps 0 --steps 3 --warmup 3 > gpurun_out/bench50_c3.log 2>&1
UP_NVCC_FLAGS="-DUP_TCW_LEAN2=0" python paper_2605_06221_b200/build.py -f > /dev/null 2>&1
for r in 1 2; do for s in gemma qwen qwen-tp8 mha gqa2 mha256; do echo "nolean2 $s $(SHAPE=$s timeout 120 python tools/score_timing.py 2>&1 | tail -1)" >> gpurun_out/score_timing50.txt; done; done
timeout 400 python bench.py --skip-cpu --config c4 --e2e-steps 0 --steps 3 --warmup 3 > gpurun_out/bench50_c4_old.log 2>&1
timeout 400 python bench.py --skip-cpu --config c3 --e2e-steps 0 --steps 3 --warmup 3 > gpurun_out/bench50_c3_old.log 2>&1
python paper_2605_06221_b200/build.py -f > /dev/null 2>&1
