# GPU box: select test across every size class, eager and graph.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_select.py -q -x > gpurun_out/pytest67.log 2>&1; echo "rc=$?" >> gpurun_out/pytest67.log
