# Dev (GPU box): fine-sampled source profiles of the latency-bound tail kernels.
set -u
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 1 --no-graph --e2e-steps 0 --skip-cpu --layer-sets 2"
timeout 300 ncu --set full --import-source on --warp-sampling-interval 0 --clock-control none -k 'regex:pair_weights|block_combine_peer' -s 2 -c 2 -o gpurun_out/prof10_c3rank -f $B --config c3-rank > gpurun_out/prof10_c3rank.log 2>&1
timeout 300 ncu --set full --import-source on --warp-sampling-interval 0 --clock-control none -k 'regex:pair_weights|block_combine|select_radix|compact_small|score_tcw' -s 5 -c 5 -o gpurun_out/prof10_c1 -f $B --config c1 > gpurun_out/prof10_c1.log 2>&1
