# Dev (GPU box): PDL families re-checked with reconstitution in the step (UP_PDL_MASK A/B).
set -u
mkdir -p gpurun_out
for r in 1 2; do for M in 11 15 27 31; do
  UP_PDL_MASK=$M timeout 300 python bench.py --skip-cpu --e2e-steps 0 --steps 5 --warmup 3 > gpurun_out/bench64.log 2>&1
  echo "c2 $r $M $(tail -n 1 gpurun_out/bench64.log | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e6,2), round(d["ms_per_step"],3))')" >> gpurun_out/pdl64.txt
done; done
for M in 11 31; do
  UP_PDL_MASK=$M timeout 400 python bench.py --skip-cpu --config c5 --e2e-steps 0 --steps 3 --warmup 3 > gpurun_out/bench64.log 2>&1
  echo "c5 $M $(tail -n 1 gpurun_out/bench64.log | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e6,2), round(d["ms_per_step"],3))')" >> gpurun_out/pdl64.txt
  UP_PDL_MASK=$M timeout 300 python bench.py --skip-cpu --config c1 --e2e-steps 0 --steps 30 --warmup 5 > gpurun_out/bench64.log 2>&1
  echo "c1 $M $(tail -n 1 gpurun_out/bench64.log | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e6,2), round(d["ms_per_step"],4))')" >> gpurun_out/pdl64.txt
done
