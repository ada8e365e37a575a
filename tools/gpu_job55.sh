# GPU box: functional N=2 runs of bench.py on one device (gloo backend; both ranks share cuda:0).
set -u
mkdir -p gpurun_out
export UP_BENCH_BACKEND=gloo
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --skip-cpu > gpurun_out/bench55_n2_c2.log 2>&1; echo "rc=$?" >> gpurun_out/bench55_n2_c2.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --config c3 --steps 3 --warmup 3 --skip-cpu > gpurun_out/bench55_n2_c3.log 2>&1; echo "rc=$?" >> gpurun_out/bench55_n2_c3.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --impl reference --steps 3 --warmup 3 > gpurun_out/bench55_n2_ref.log 2>&1; echo "rc=$?" >> gpurun_out/bench55_n2_ref.log
