# GPU box: launch lists (cold, serialised per-launch times) of c1 and c3-rank on the final kernels.
set -u
mkdir -p gpurun_out
for C in c1 c3-rank; do
ncu --kernel-name regex:"score|pair_weights|combine|select|expand|compact|scatter|peer" --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches60_$C.csv \
  python bench.py --config $C --steps 1 --warmup 1 --no-graph --e2e-steps 0 --skip-cpu --layer-sets 2 > gpurun_out/launches60_$C.log 2>&1
done
