# Dev (GPU box): pair_weights CTA size at C1 (8 warps default) and c3-rank (32).
set -u
mkdir -p gpurun_out
for r in 1 2; do for w in 0 4 16 32; do
  UP_PW_WARPS=$w timeout 300 python bench.py --skip-cpu --config c1 --e2e-steps 0 --steps 30 --warmup 5 > gpurun_out/bench54_c1.log 2>&1
  echo "c1 $r $w $(tail -n 1 gpurun_out/bench54_c1.log | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e6,1), d["stages"]["score"]["ms_per_layer"]*1e3)')" >> gpurun_out/pw_54.txt
done; done
for w in 0 8 16; do
  UP_PW_WARPS=$w timeout 300 python bench.py --skip-cpu --config c3-rank --e2e-steps 0 --steps 3 --warmup 3 > gpurun_out/bench54_c3r.log 2>&1
  echo "c3rank $w $(tail -n 1 gpurun_out/bench54_c3r.log | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e6,1), d["stages"]["score"]["ms_per_layer"]*1e3)')" >> gpurun_out/pw_54.txt
done
