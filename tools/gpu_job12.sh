# Dev (GPU box): full GPU suite + smoke + key benches on the current tree.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest12.log 2>&1; echo "rc=$?" >> gpurun_out/pytest12.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke12.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke12.log
python tools/select_timing.py > gpurun_out/select_timing12.txt 2>&1
for c in c1 c2 c3-rank; do timeout 300 python bench.py --skip-cpu --config $c --e2e-steps 0 > gpurun_out/bench12_$c.log 2>&1; done
B="python bench.py --steps 1 --warmup 1 --no-graph --e2e-steps 0 --skip-cpu --layer-sets 2"
K='regex:score|select|compact|pair_|block_combine|expand|scatter|slot|peer'
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -c 16 --csv --log-file gpurun_out/launches12_c1.csv $B --config c1 > /dev/null 2>&1
