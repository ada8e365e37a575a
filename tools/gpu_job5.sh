# Dev (GPU box): full GPU suite after radix select + SPLIT heuristic; bench modes; TP N=2 functional.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest5.log 2>&1; echo "rc=$?" >> gpurun_out/pytest5.log
python tools/select_timing.py > gpurun_out/select_timing5.txt 2>&1
timeout 400 python bench.py --skip-cpu > gpurun_out/bench5_c2.log 2>&1
timeout 400 python bench.py --skip-cpu --config c1 > gpurun_out/bench5_c1.log 2>&1
timeout 400 python bench.py --skip-cpu --config c3-rank > gpurun_out/bench5_c3rank.log 2>&1
timeout 400 python bench.py --skip-cpu --config c4 --e2e-steps 1 > gpurun_out/bench5_c4.log 2>&1
timeout 400 python bench.py --skip-cpu --config c5 --e2e-steps 0 > gpurun_out/bench5_c5.log 2>&1
UP_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --config c3 --steps 2 --warmup 1 --e2e-steps 0 > gpurun_out/bench5_tp2.log 2>&1
UP_NVCC_FLAGS="-DUP_SELECT_ALWAYS_SORT" python paper_2605_06221_b200/build.py -f > /dev/null 2>&1
echo "--- always sort" >> gpurun_out/select_timing5.txt
python tools/select_timing.py >> gpurun_out/select_timing5.txt 2>&1
python paper_2605_06221_b200/build.py -f > /dev/null 2>&1
