set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 400 python bench.py > gpurun_out/bench_c2.log 2>&1
for c in c1 c3 c4 c5; do timeout 400 python bench.py --config $c --skip-cpu > gpurun_out/bench_$c.log 2>&1; done
timeout 400 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1
OUT=gpurun_out timeout 900 bash profiles/run_profile.sh > gpurun_out/run_profile.log 2>&1
