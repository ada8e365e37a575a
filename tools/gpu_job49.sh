# Dev (GPU box): pair_weights warp path vs CTA path bitwise.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scorer.py tests/test_gpu_peer.py -x -q > gpurun_out/pytest49.log 2>&1; echo "rc=$?" >> gpurun_out/pytest49.log
