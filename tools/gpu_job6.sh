# Dev (GPU box): radix select v2 A/B + parity; small-capacity fused paths (c1); c3-rank launch list.
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_select.py tests/test_gpu_acceptance.py tests/test_gpu_compact.py tests/test_gpu_golden_e2e.py tests/test_gpu_scorer.py -x -q > gpurun_out/pytest6.log 2>&1; echo "rc=$?" >> gpurun_out/pytest6.log
python tools/select_timing.py > gpurun_out/select_timing6.txt 2>&1
timeout 300 python bench.py --skip-cpu --config c1 > gpurun_out/bench6_c1.log 2>&1
timeout 300 python bench.py --skip-cpu --e2e-steps 0 > gpurun_out/bench6_c2.log 2>&1
timeout 300 python bench.py --skip-cpu --config c3-rank --e2e-steps 0 > gpurun_out/bench6_c3rank.log 2>&1
B="python bench.py --steps 1 --warmup 1 --no-graph --e2e-steps 0 --skip-cpu --layer-sets 2"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches6_c1.csv $B --config c1 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches6_c3rank.csv $B --config c3-rank > /dev/null 2>&1
UP_NVCC_FLAGS="-DUP_SELECT_ALWAYS_SORT" python paper_2605_06221_b200/build.py -f > /dev/null 2>&1
echo "--- always sort" >> gpurun_out/select_timing6.txt
python tools/select_timing.py >> gpurun_out/select_timing6.txt 2>&1
timeout 300 python bench.py --skip-cpu --e2e-steps 0 > gpurun_out/bench6_c2_sort.log 2>&1
python paper_2605_06221_b200/build.py -f > /dev/null 2>&1
