# Dev (GPU box): small compaction with fewer CTAs per SM (2, 3 vs 4) at C1.
set -u
mkdir -p gpurun_out
for r in 1 2; do for n in 2 3 4; do
  UP_SMALL_COMPACT_CTAS_PER_SM=$n timeout 300 python bench.py --skip-cpu --config c1 --e2e-steps 0 --steps 30 --warmup 5 > gpurun_out/bench53_c1_$n.log 2>&1
  echo "$r $n $(tail -n 1 gpurun_out/bench53_c1_$n.log | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e6,1), d["stages"]["compact"]["ms_per_layer"]*1e3)')" >> gpurun_out/c1_53.txt
done; done
