# Dev (GPU box): tiny select path A/B + phase stamps.
set -u
mkdir -p gpurun_out
python tools/select_timing.py > gpurun_out/select22_tiny.txt 2>&1
timeout 120 python tools/select_phases.py > gpurun_out/select22_phases_tiny.txt 2>&1
timeout 300 python bench.py --skip-cpu --config c1 --e2e-steps 0 > gpurun_out/bench22_c1_tiny.log 2>&1
UP_NVCC_FLAGS="-DUP_TINY_SELECT=1" python paper_2605_06221_b200/build.py -f > /dev/null 2>&1
python tools/select_timing.py > gpurun_out/select22_notiny.txt 2>&1
timeout 120 python tools/select_phases.py > gpurun_out/select22_phases_notiny.txt 2>&1
timeout 300 python bench.py --skip-cpu --config c1 --e2e-steps 0 > gpurun_out/bench22_c1_notiny.log 2>&1
python paper_2605_06221_b200/build.py -f > /dev/null 2>&1
