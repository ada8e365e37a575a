# GPU box: sanitizer pass after the late round-2 changes + bench lines with the new score-stage bounds.
set -u
mkdir -p gpurun_out
bash tools/gpu_sanitize.sh
timeout 300 python bench.py --skip-cpu --config c3-rank --e2e-steps 0 --steps 3 --warmup 3 > gpurun_out/bench46_c3rank.log 2>&1
timeout 300 python bench.py --skip-cpu --config c1 --e2e-steps 0 --steps 20 --warmup 5 > gpurun_out/bench46_c1.log 2>&1
