set -u
mkdir -p gpurun_out
python tools/debug_hpc1b.py > gpurun_out/debug30.txt 2>&1
UP_NVCC_FLAGS="-DUP_TCW_POLY_PAIRS_D128=0" python paper_2605_06221_b200/build.py -f > /dev/null 2>&1
echo "--- NP=0" >> gpurun_out/debug30.txt; python tools/debug_hpc1b.py >> gpurun_out/debug30.txt 2>&1
UP_NVCC_FLAGS="-DUP_TCW_LEAN=0" python paper_2605_06221_b200/build.py -f > /dev/null 2>&1
echo "--- LEAN=0" >> gpurun_out/debug30.txt; python tools/debug_hpc1b.py >> gpurun_out/debug30.txt 2>&1
python paper_2605_06221_b200/build.py -f > /dev/null 2>&1
