# GPU box: scorer parity matrix with the added own-subtile cases.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scorer.py -q -x -k "tc_scorer_matches_oracle" > gpurun_out/pytest66.log 2>&1; echo "rc=$?" >> gpurun_out/pytest66.log
