# GPU box: compute-sanitizer over the round-2 kernels (memcheck / synccheck / racecheck).
set -u
mkdir -p gpurun_out
CS="compute-sanitizer --print-limit 20"
S="gpurun_out/sanitizer_r02.txt"
: > $S
run() { echo "=== $*" >> $S; timeout 1200 "$@" >> $S 2>&1; echo "rc=$?" >> $S; }
run $CS --tool memcheck python -c 'import __graft_entry__ as g; g.smoke()'
run $CS --tool memcheck python -m pytest -q -x tests/test_gpu_select.py tests/test_gpu_compact.py
run $CS --tool memcheck python -m pytest -q -x tests/test_gpu_scorer.py -k "not variants"
run $CS --tool memcheck python -m pytest -q -x tests/test_gpu_golden_e2e.py
run $CS --tool synccheck python -c 'import __graft_entry__ as g; g.smoke()'
run $CS --tool racecheck python -m pytest -q -x tests/test_gpu_select.py -k "worked or random or varlen or c3_sample"
run $CS --tool racecheck python -m pytest -q -x tests/test_gpu_compact.py -k small_capacity
run $CS --tool racecheck python -m pytest -q -x tests/test_gpu_scorer.py -k "many_requests"
