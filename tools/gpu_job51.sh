# Dev (GPU box): c2 scorer knobs re-checked on the final code: SPLIT epilogue, SUBN=64 for HPC 4.
set -u
mkdir -p gpurun_out
for r in 1 2; do
  echo "default $(SHAPE=llama timeout 120 python tools/score_timing.py 2>&1 | tail -1)" >> gpurun_out/score_timing51.txt
  echo "split $(UP_TCW_SPLIT=1 SHAPE=llama timeout 120 python tools/score_timing.py 2>&1 | tail -1)" >> gpurun_out/score_timing51.txt
done
UP_NVCC_FLAGS="-DUP_TCW_SUBN_HPC4=64" python paper_2605_06221_b200/build.py -f > /dev/null 2>&1
for r in 1 2; do echo "subn64 $(SHAPE=llama timeout 120 python tools/score_timing.py 2>&1 | tail -1)" >> gpurun_out/score_timing51.txt; done
python paper_2605_06221_b200/build.py -f > /dev/null 2>&1
