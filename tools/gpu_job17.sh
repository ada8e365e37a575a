# Dev (GPU box): query tiles (n > 128 on tensor cores) + unified combine arithmetic.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest17.log 2>&1; echo "rc=$?" >> gpurun_out/pytest17.log
for n in 128 256 512; do timeout 600 python bench.py --skip-cpu --e2e-steps 0 --query-window $n > gpurun_out/bench17_c2_n$n.log 2>&1; done
timeout 600 python bench.py --skip-cpu --e2e-steps 0 --config c3 --query-window 512 > gpurun_out/bench17_c3_n512.log 2>&1
