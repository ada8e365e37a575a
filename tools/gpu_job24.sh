# Dev (GPU box): per-head Q barriers + (row, plane) small compaction.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest24.log 2>&1; echo "rc=$?" >> gpurun_out/pytest24.log
LENGTHS=4096 timeout 120 python tools/score_phases.py > gpurun_out/score_phases24.txt 2>&1
for s in llama4k llama gemma qwen; do echo "$s $(SHAPE=$s timeout 120 python tools/score_timing.py 2>&1 | tail -1)" >> gpurun_out/score_timing24.txt; done
timeout 300 python bench.py --skip-cpu --config c1 --e2e-steps 0 > gpurun_out/bench24_c1.log 2>&1
timeout 300 python bench.py --skip-cpu --e2e-steps 0 > gpurun_out/bench24_c2.log 2>&1
