# Dev (GPU box): filtered launch lists for c1 / c3-rank; scorer tests after the SIMT fallback.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scorer.py tests/test_gpu_select.py tests/test_gpu_compact.py -x -q > gpurun_out/pytest7.log 2>&1; echo "rc=$?" >> gpurun_out/pytest7.log
B="python bench.py --steps 1 --warmup 1 --no-graph --e2e-steps 0 --skip-cpu --layer-sets 2"
K='regex:score|select|compact|pair_|block_combine|expand|scatter|slot|peer'
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -c 40 --csv --log-file gpurun_out/launches7_c1.csv $B --config c1 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -c 40 --csv --log-file gpurun_out/launches7_c3rank.csv $B --config c3-rank > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k 'regex:score_tcw|block_combine_peer|pair_w' -s 3 -c 3 -o gpurun_out/prof7_c3rank -f $B --config c3-rank > gpurun_out/prof7_c3rank.log 2>&1
