# Dev (GPU box): pair_weights candidate enumeration; first-subtile A/B.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scorer.py tests/test_gpu_golden_e2e.py tests/test_gpu_peer.py -x -q > gpurun_out/pytest40.log 2>&1; echo "rc=$?" >> gpurun_out/pytest40.log
for r in 1 2; do for s in llama llama4k gemma mha mixed-llama; do echo "first $s $(SHAPE=$s timeout 120 python tools/score_timing.py 2>&1 | tail -1)" >> gpurun_out/score_timing40.txt; done; done
UP_NVCC_FLAGS="-DUP_TCW_FIRST_REF=0" python paper_2605_06221_b200/build.py -f > /dev/null 2>&1
for r in 1 2; do for s in llama llama4k gemma mha mixed-llama; do echo "nofirst $s $(SHAPE=$s timeout 120 python tools/score_timing.py 2>&1 | tail -1)" >> gpurun_out/score_timing40.txt; done; done
python paper_2605_06221_b200/build.py -f > /dev/null 2>&1
for s in mixed mixed-llama; do
SHAPE=$s timeout 300 ncu --kernel-name regex:"score|pair_weights|block_combine|plan" --metrics gpu__time_duration.sum --clock-control none -c 12 --csv --log-file gpurun_out/ncu40_$s.csv python tools/score_timing.py > /dev/null 2>&1
done
