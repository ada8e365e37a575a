# Dev (GPU box): many short requests -- where does the scorer stage spend its time?
set -u
mkdir -p gpurun_out
for s in mixed mixed-llama; do
SHAPE=$s timeout 300 ncu --kernel-name regex:"score|pair_weights|block_combine|plan" --metrics gpu__time_duration.sum --clock-control none -c 12 --csv --log-file gpurun_out/ncu38_$s.csv python tools/score_timing.py > /dev/null 2>&1
done
