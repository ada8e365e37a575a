# Dev (GPU box): score_tcw HPC=1 after the statistics-sizing fix -- full suite + timings.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest33.log 2>&1; echo "rc=$?" >> gpurun_out/pytest33.log
for s in mha mha256 llama gemma qwen; do echo "$s $(SHAPE=$s timeout 120 python tools/score_timing.py 2>&1 | tail -1)" >> gpurun_out/score_timing33.txt; done
for n in 32 64; do timeout 600 python bench.py --skip-cpu --e2e-steps 0 --query-window $n > gpurun_out/bench33_c2_n$n.log 2>&1; done
timeout 600 python bench.py --skip-cpu --e2e-steps 0 > gpurun_out/bench33_c2.log 2>&1
