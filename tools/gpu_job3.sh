# Dev (GPU box): ncu of the CTA-pair scorer (UP_TC2=1) on the c2 shape.
set -u
mkdir -p gpurun_out
BENCH="python bench.py --config c2 --steps 1 --warmup 1 --no-graph --e2e-steps 0 --skip-cpu --layer-sets 2"
UP_TC2=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:'score_tc2' -s 4 -c 1 \
    -o gpurun_out/prof_tc2 -f $BENCH > gpurun_out/prof_tc2.log 2>&1
