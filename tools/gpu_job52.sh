# Dev (GPU box): DRAM bytes of the D = 256 scorers (c3 TP group, c4 Gemma) vs their K-stream bytes.
set -u
mkdir -p gpurun_out
for s in qwen-tp8 gemma qwen; do
SHAPE=$s timeout 300 ncu --kernel-name regex:"score_tcw" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none -c 3 --csv --log-file gpurun_out/ncu52_$s.csv python tools/score_timing.py > /dev/null 2>&1
done
