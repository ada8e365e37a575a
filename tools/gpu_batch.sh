set -u
# Round-end check on the GPU box: tests, smoke, bench c1-c5 (+ c3-rank, c5-mixed, stacked
# c2), the reference arm, profiles.  The ncu reports are summarised on the box
# (profiles/summarize.py) and only the summaries come back (gpurun_out/ is capped at 64 MiB).
TAG=${TAG:-r02}
mkdir -p gpurun_out/summ
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 400 python bench.py > gpurun_out/bench_c2.log 2>&1
for c in c1 c3 c3-rank c4 c5 c5-mixed; do timeout 400 python bench.py --config $c --skip-cpu > gpurun_out/bench_$c.log 2>&1; done
timeout 400 python bench.py --stack 2 --skip-cpu --e2e-steps 0 > gpurun_out/bench_c2_stack2.log 2>&1
timeout 400 python bench.py --regime iid --skip-cpu --e2e-steps 0 > gpurun_out/bench_c2_iid.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1
if [ "${PROFILE:-1}" = "1" ]; then
  for C in ${PROFILE_CONFIGS:-c2}; do
    T=$([ "$C" = "c2" ] && echo "" || echo "_$C")
    OUT=gpurun_out CONFIG=$C TAG=$T timeout 900 bash profiles/run_profile.sh > gpurun_out/run_profile$T.log 2>&1
    python profiles/summarize.py gpurun_out $TAG "$T" $C > /dev/null 2>&1
    cp profiles/ncu_summary_$TAG$T.md profiles/launches_$TAG$T.csv gpurun_out/summ/ 2>/dev/null
    rm -f gpurun_out/*.ncu-rep
  done
  cp profiles/ncu_traffic.json gpurun_out/summ/ 2>/dev/null
fi
