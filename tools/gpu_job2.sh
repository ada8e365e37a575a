# Dev (GPU box): scorer profile (ncu full + source) and exp2/poly sweeps.
set -u
mkdir -p gpurun_out tools/_bin
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -o tools/_bin/ubench_ex2 tools/ubench_ex2.cu && tools/_bin/ubench_ex2 g > gpurun_out/ubench_group.txt 2>&1
BENCH="python bench.py --config c2 --steps 1 --warmup 1 --no-graph --e2e-steps 0 --skip-cpu --layer-sets 2"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'score_tcw|pair_weights|block_combine' -s 6 -c 3 \
    -o gpurun_out/prof_score -f $BENCH > gpurun_out/prof_score.log 2>&1
for P in 4 6 8 10; do
  UP_NVCC_FLAGS="-DUP_TCW_POLY_PAIRS_D128=$P" python paper_2605_06221_b200/build.py -f > /dev/null 2>&1
  echo "P=$P $(timeout 120 python tools/score_timing.py 2>&1 | tail -1) | iid $(REGIME=iid timeout 120 python tools/score_timing.py 2>&1 | tail -1)" >> gpurun_out/poly_sweep.txt
done
python paper_2605_06221_b200/build.py -f > /dev/null 2>&1
