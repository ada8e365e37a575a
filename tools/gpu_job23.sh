# Dev (GPU box): select without the tiny path + faster fused expansion.
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_select.py tests/test_gpu_compact.py tests/test_gpu_golden_e2e.py tests/test_gpu_acceptance.py tests/test_gpu_cascade.py -q > gpurun_out/pytest23.log 2>&1; echo "rc=$?" >> gpurun_out/pytest23.log
python tools/select_timing.py > gpurun_out/select23.txt 2>&1
timeout 120 python tools/select_phases.py > gpurun_out/select23_phases.txt 2>&1
timeout 300 python bench.py --skip-cpu --config c1 > gpurun_out/bench23_c1.log 2>&1
