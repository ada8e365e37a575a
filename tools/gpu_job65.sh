# GPU box: bench contract test + a default bench line after the roofline "also" field.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bench_contract.py -q -x > gpurun_out/pytest65.log 2>&1; echo "rc=$?" >> gpurun_out/pytest65.log
timeout 400 python bench.py --steps 5 --warmup 3 > gpurun_out/bench65_c2.log 2>&1
