# Dev (GPU box): radix select v2 in the 512-thread class (A/B), full GPU suite on the current tree.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest21.log 2>&1; echo "rc=$?" >> gpurun_out/pytest21.log
python tools/select_timing.py > gpurun_out/select21_default.txt 2>&1
for c in c3 c4 c5; do timeout 300 python bench.py --skip-cpu --e2e-steps 0 --config $c --steps 2 --warmup 1 > gpurun_out/bench21_${c}_default.log 2>&1; done
UP_NVCC_FLAGS="-DUP_SELECT_RADIX_MAX_THREADS=512" python paper_2605_06221_b200/build.py -f > /dev/null 2>&1
python tools/select_timing.py > gpurun_out/select21_radix512.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_select.py tests/test_gpu_acceptance.py -q > gpurun_out/pytest21_radix512.log 2>&1; echo "rc=$?" >> gpurun_out/pytest21_radix512.log
for c in c3 c4 c5; do timeout 300 python bench.py --skip-cpu --e2e-steps 0 --config $c --steps 2 --warmup 1 > gpurun_out/bench21_${c}_radix512.log 2>&1; done
python paper_2605_06221_b200/build.py -f > /dev/null 2>&1
