# GPU box: c3-rank bench line on the final kernels (peer combine at 32 warps per CTA).
set -u
mkdir -p gpurun_out
timeout 400 python bench.py --config c3-rank --skip-cpu > gpurun_out/bench_c3-rank.log 2>&1
timeout 600 python -m pytest tests/test_gpu_peer.py tests/test_gpu_scorer.py -q -x -k "tp or peer or shards" > gpurun_out/pytest62.log 2>&1; echo "rc=$?" >> gpurun_out/pytest62.log
