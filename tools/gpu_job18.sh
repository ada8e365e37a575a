# Dev (GPU box): row packing (n <= 64) + n=512 full-size parity.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_scorer.py tests/test_gpu_golden_e2e.py tests/test_gpu_select.py tests/test_gpu_peer.py "tests/test_gpu_fullsize.py::test_llama_32k_query_window_512" -q > gpurun_out/pytest18.log 2>&1; echo "rc=$?" >> gpurun_out/pytest18.log
for n in 32 64; do timeout 600 python bench.py --skip-cpu --e2e-steps 0 --query-window $n > gpurun_out/bench18_c2_n$n.log 2>&1; done
UP_NO_QPACK=1 timeout 600 python bench.py --skip-cpu --e2e-steps 0 --query-window 64 > gpurun_out/bench18_c2_n64_nopack.log 2>&1
timeout 600 python bench.py --skip-cpu --e2e-steps 0 --config c3 --query-window 32 > gpurun_out/bench18_c3_n32.log 2>&1
