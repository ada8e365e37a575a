# Dev (GPU box): pair_weights warp path + no wasted first-subtile pass in score_tcw.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scorer.py tests/test_gpu_golden_e2e.py tests/test_gpu_peer.py tests/test_gpu_cascade.py -x -q > gpurun_out/pytest39.log 2>&1; echo "rc=$?" >> gpurun_out/pytest39.log
for s in llama llama4k gemma qwen mha mixed mixed-llama short-mha; do echo "$s $(SHAPE=$s timeout 120 python tools/score_timing.py 2>&1 | tail -1)" >> gpurun_out/score_timing39.txt; done
timeout 300 python bench.py --skip-cpu --config c1 --steps 20 --warmup 5 > gpurun_out/bench39_c1.log 2>&1
for s in mixed mixed-llama; do
SHAPE=$s timeout 300 ncu --kernel-name regex:"score|pair_weights|block_combine|plan" --metrics gpu__time_duration.sum --clock-control none -c 12 --csv --log-file gpurun_out/ncu39_$s.csv python tools/score_timing.py > /dev/null 2>&1
done
