# Dev (GPU box): SPLIT epilogue A/B + parity, cascaded bench modes.
set -u
mkdir -p gpurun_out
for s in llama llama4k; do
  echo "split $(SHAPE=$s timeout 120 python tools/score_timing.py 2>&1 | tail -1)" >> gpurun_out/split_timing.txt
  echo "nosplit $(UP_TCW_SPLIT=0 SHAPE=$s timeout 120 python tools/score_timing.py 2>&1 | tail -1)" >> gpurun_out/split_timing.txt
  echo "split-iid $(REGIME=iid SHAPE=$s timeout 120 python tools/score_timing.py 2>&1 | tail -1)" >> gpurun_out/split_timing.txt
done
timeout 900 python -m pytest tests/test_gpu_scorer.py tests/test_gpu_golden_e2e.py tests/test_gpu_fullsize.py tests/test_gpu_acceptance.py -x -q > gpurun_out/pytest_split.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_split.log
timeout 400 python bench.py --skip-cpu > gpurun_out/bench4_c2.log 2>&1
timeout 400 python bench.py --skip-cpu --config c3-rank > gpurun_out/bench4_c3rank.log 2>&1
timeout 400 python bench.py --skip-cpu --config c4 > gpurun_out/bench4_c4.log 2>&1
timeout 400 python bench.py --skip-cpu --stack 2 --e2e-steps 0 > gpurun_out/bench4_c2s2.log 2>&1
timeout 400 python bench.py --skip-cpu --config c3 --e2e-steps 0 > gpurun_out/bench4_c3.log 2>&1
