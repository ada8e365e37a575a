# Dev (GPU box): small compaction grid (CTAs per SM) A/B at C1; compaction tests.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_compact.py tests/test_gpu_golden_e2e.py -x -q > gpurun_out/pytest45.log 2>&1; echo "rc=$?" >> gpurun_out/pytest45.log
for r in 1 2; do for n in 4 6 8 12; do
  UP_SMALL_COMPACT_CTAS_PER_SM=$n timeout 300 python bench.py --skip-cpu --config c1 --e2e-steps 0 --steps 20 --warmup 5 > gpurun_out/bench45_c1_$n.log 2>&1
  echo "$r $n $(tail -n 1 gpurun_out/bench45_c1_$n.log | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e6,1), d["stages"]["compact"]["ms_per_layer"]*1e3, d["stages"]["select"]["us_per_event"], d["stages"]["score"]["ms_per_layer"]*1e3)')" >> gpurun_out/c1_45.txt
done; done
