# Dev (GPU box): in-scorer pair merge (no pair_weights launch) -- full GPU suite + timings.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest11.log 2>&1; echo "rc=$?" >> gpurun_out/pytest11.log
for s in llama llama4k gemma qwen qwen-tp8; do
  echo "fused $(SHAPE=$s timeout 120 python tools/score_timing.py 2>&1 | tail -1)" >> gpurun_out/score_timing11.txt
  echo "kernel $(UP_PAIR_WEIGHTS_KERNEL=1 SHAPE=$s timeout 120 python tools/score_timing.py 2>&1 | tail -1)" >> gpurun_out/score_timing11.txt
done
for c in c1 c2 c3-rank c4; do timeout 300 python bench.py --skip-cpu --config $c --e2e-steps 0 > gpurun_out/bench11_$c.log 2>&1; done
B="python bench.py --steps 1 --warmup 1 --no-graph --e2e-steps 0 --skip-cpu --layer-sets 2"
K='regex:score|select|compact|pair_|block_combine|expand|scatter|slot|peer'
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -c 16 --csv --log-file gpurun_out/launches11_c3rank.csv $B --config c3-rank > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -c 16 --csv --log-file gpurun_out/launches11_c1.csv $B --config c1 > /dev/null 2>&1
