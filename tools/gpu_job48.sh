# Dev (GPU box): small compaction with split rows (A/B UP_SMALL_COPY_SPLIT).
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_compact.py tests/test_gpu_golden_e2e.py tests/test_gpu_cascade.py -x -q > gpurun_out/pytest48.log 2>&1; echo "rc=$?" >> gpurun_out/pytest48.log
for r in 1 2; do
  timeout 300 python bench.py --skip-cpu --config c1 --steps 20 --warmup 5 > gpurun_out/bench48_c1_split.log 2>&1
  echo "split $(tail -n 1 gpurun_out/bench48_c1_split.log | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e6,1), d["stages"]["compact"]["ms_per_layer"]*1e3, d["e2e"]["value"]/1e6)')" >> gpurun_out/c1_48.txt
done
UP_NVCC_FLAGS="-DUP_SMALL_COPY_SPLIT=0" python paper_2605_06221_b200/build.py -f > /dev/null 2>&1
for r in 1 2; do
  timeout 300 python bench.py --skip-cpu --config c1 --e2e-steps 0 --steps 20 --warmup 5 > gpurun_out/bench48_c1_nosplit.log 2>&1
  echo "nosplit $(tail -n 1 gpurun_out/bench48_c1_nosplit.log | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e6,1), d["stages"]["compact"]["ms_per_layer"]*1e3)')" >> gpurun_out/c1_48.txt
done
python paper_2605_06221_b200/build.py -f > /dev/null 2>&1
