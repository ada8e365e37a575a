# Dev (GPU box): pair_weights range table + acq_rel peer fence.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scorer.py tests/test_gpu_golden_e2e.py tests/test_gpu_peer.py -x -q > gpurun_out/pytest9.log 2>&1; echo "rc=$?" >> gpurun_out/pytest9.log
B="python bench.py --steps 1 --warmup 1 --no-graph --e2e-steps 0 --skip-cpu --layer-sets 2"
K='regex:score|select|compact|pair_|block_combine|expand|scatter|slot|peer'
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -c 20 --csv --log-file gpurun_out/launches9_c3rank.csv $B --config c3-rank > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -c 20 --csv --log-file gpurun_out/launches9_c2.csv $B --config c2 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -c 20 --csv --log-file gpurun_out/launches9_c1.csv $B --config c1 > /dev/null 2>&1
timeout 300 python bench.py --skip-cpu --config c3-rank --e2e-steps 0 > gpurun_out/bench9_c3rank.log 2>&1
timeout 300 python bench.py --skip-cpu --e2e-steps 0 > gpurun_out/bench9_c2.log 2>&1
