# Dev (GPU box): full ncu capture of the HPC 1 (MHA) and HPC 4 (LLaMA) scorers with source, summarised on the box.
set -u
mkdir -p gpurun_out
for s in mha llama; do
SHAPE=$s timeout 600 ncu --set full --import-source on --clock-control none --kernel-name regex:"score_tcw" -c 1 -o gpurun_out/ncu56_$s python tools/score_timing.py > gpurun_out/ncu56_$s.log 2>&1
python profiles/stall_summary.py gpurun_out/ncu56_$s.ncu-rep score_tcw 25 > gpurun_out/ncu56_$s.md 2>&1
ncu -i gpurun_out/ncu56_$s.ncu-rep --page raw --csv > gpurun_out/ncu56_${s}_raw.csv 2>/dev/null
rm -f gpurun_out/ncu56_$s.ncu-rep
done
