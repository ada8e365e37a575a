# Dev (GPU box): scorer stage time for prebuilt library variants in tools/_bin/var/*.so
cp paper_2605_06221_b200/_lib/libuniprefill_b200.so /tmp/orig.so
for f in tools/_bin/var/*.so; do
  n=$(basename $f .so)
  cp $f paper_2605_06221_b200/_lib/libuniprefill_b200.so
  echo "$n $(SHAPE=${SHAPE:-llama} timeout 120 python tools/score_timing.py) | $(SHAPE=${SHAPE:-llama} timeout 120 python tools/score_timing.py)"
done >> gpurun_out/diag.txt 2>&1
cp /tmp/orig.so paper_2605_06221_b200/_lib/libuniprefill_b200.so
