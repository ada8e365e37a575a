# Dev (GPU box): peer-fused combine CTA size at c3-rank (and TP peer tests).
set -u
mkdir -p gpurun_out
for T in 512 1024; do UP_PEER_COMBINE_THREADS=$T timeout 600 python -m pytest tests/test_gpu_peer.py -x -q > gpurun_out/pytest61_$T.log 2>&1; echo "rc=$?" >> gpurun_out/pytest61_$T.log; done
for r in 1 2; do for T in 256 512 1024; do
  UP_PEER_COMBINE_THREADS=$T timeout 300 python bench.py --skip-cpu --config c3-rank --e2e-steps 0 --steps 3 --warmup 3 > gpurun_out/bench61.log 2>&1
  echo "$r $T $(tail -n 1 gpurun_out/bench61.log | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e6,1), d["stages"]["score"]["ms_per_layer"]*1e3)')" >> gpurun_out/peer61.txt
done; done
