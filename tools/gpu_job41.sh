# Dev (GPU box): pair_weights warp task = pair.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scorer.py tests/test_gpu_golden_e2e.py tests/test_gpu_peer.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest41.log 2>&1; echo "rc=$?" >> gpurun_out/pytest41.log
for s in llama llama4k qwen mixed mixed-llama; do echo "$s $(SHAPE=$s timeout 120 python tools/score_timing.py 2>&1 | tail -1)" >> gpurun_out/score_timing41.txt; done
for s in mixed-llama llama4k; do
SHAPE=$s timeout 300 ncu --kernel-name regex:"score|pair_weights|block_combine|plan" --metrics gpu__time_duration.sum --clock-control none -c 12 --csv --log-file gpurun_out/ncu41_$s.csv python tools/score_timing.py > /dev/null 2>&1
done
