# Dev (GPU box): select brute-force ranks for <= 128 blocks (A/B), scorer PDL prologue,
# small-compaction unroll; exp2 roofline in bench.
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_select.py tests/test_gpu_golden_e2e.py tests/test_gpu_compact.py tests/test_gpu_scorer.py tests/test_gpu_acceptance.py -x -q > gpurun_out/pytest42.log 2>&1; echo "rc=$?" >> gpurun_out/pytest42.log
echo "brute" >> gpurun_out/select42.txt; timeout 120 python tools/select_timing.py >> gpurun_out/select42.txt 2>&1
timeout 300 python bench.py --skip-cpu --config c1 --steps 20 --warmup 5 > gpurun_out/bench42_c1.log 2>&1
timeout 300 python bench.py --skip-cpu --e2e-steps 0 --steps 5 --warmup 3 > gpurun_out/bench42_c2.log 2>&1
UP_NVCC_FLAGS="-DUP_SELECT_BRUTE=0 -DUP_SMALL_COPY_UNROLL=8" python paper_2605_06221_b200/build.py -f > /dev/null 2>&1
echo "radix" >> gpurun_out/select42.txt; timeout 120 python tools/select_timing.py >> gpurun_out/select42.txt 2>&1
timeout 300 python bench.py --skip-cpu --config c1 --steps 20 --warmup 5 > gpurun_out/bench42_c1_old.log 2>&1
python paper_2605_06221_b200/build.py -f > /dev/null 2>&1
