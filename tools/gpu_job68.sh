set -u
mkdir -p gpurun_out
for L in 3000,100 60000,3000 150000,3000 150000,60000,3000,100,1; do
  python tools/debug_select_graph.py $L >> gpurun_out/dbg68.txt 2>&1
  UP_SELECT_FORK=0 python tools/debug_select_graph.py $L >> gpurun_out/dbg68.txt 2>&1
done
