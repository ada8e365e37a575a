# GPU box: memcheck / racecheck over the last kernel changes (own-subtile walk, peer combine CTA size).
set -u
mkdir -p gpurun_out
CS="compute-sanitizer --print-limit 20"
S="gpurun_out/sanitizer_late_r02.txt"
: > $S
run() { echo "=== $*" >> $S; timeout 1500 "$@" >> $S 2>&1; echo "rc=$?" >> $S; }
run $CS --tool memcheck python -m pytest -q -x tests/test_gpu_scorer.py -k "not variants"
run $CS --tool memcheck python -m pytest -q -x tests/test_gpu_peer.py
run $CS --tool racecheck python -m pytest -q -x tests/test_gpu_scorer.py -k "many_requests or bitwise"
