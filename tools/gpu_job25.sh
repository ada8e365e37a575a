# Dev (GPU box): TMEM read throughput probe + scorer timings.
set -u
mkdir -p gpurun_out tools/_bin
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -I paper_2605_06221_b200/csrc -I include -o tools/_bin/ubench_tmem tools/ubench_tmem.cu && tools/_bin/ubench_tmem > gpurun_out/ubench_tmem.txt 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv >> gpurun_out/ubench_tmem.txt
for s in llama4k llama gemma qwen; do echo "$s $(SHAPE=$s timeout 120 python tools/score_timing.py 2>&1 | tail -1)" >> gpurun_out/score_timing25.txt; done
