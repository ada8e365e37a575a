# Dev (GPU box): cascade parity test + C1 scorer phase clocks.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cascade.py tests/test_gpu_scorer.py -q > gpurun_out/pytest19.log 2>&1; echo "rc=$?" >> gpurun_out/pytest19.log
for L in 4096 32768,32768,32768,32768; do LENGTHS=$L timeout 120 python tools/score_phases.py >> gpurun_out/score_phases19.txt 2>&1; done
