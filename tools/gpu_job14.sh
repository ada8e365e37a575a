# Dev (GPU box): chunked combine + tiny select parity/timing; PDL mask A/B for compaction.
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_scorer.py tests/test_gpu_select.py tests/test_gpu_golden_e2e.py tests/test_gpu_acceptance.py tests/test_gpu_fullsize.py -q > gpurun_out/pytest14.log 2>&1; echo "rc=$?" >> gpurun_out/pytest14.log
for s in llama llama4k gemma; do
  echo "chunked $(SHAPE=$s timeout 120 python tools/score_timing.py 2>&1 | tail -1)" >> gpurun_out/score_timing14.txt
  echo "warp $(UP_COMBINE_CHUNKED=0 SHAPE=$s timeout 120 python tools/score_timing.py 2>&1 | tail -1)" >> gpurun_out/score_timing14.txt
done
timeout 120 python tools/select_phases.py > gpurun_out/select_phases14.txt 2>&1
timeout 120 python tools/score_phases.py > gpurun_out/score_phases14.txt 2>&1
for m in 11 27 15 31; do UP_PDL_MASK=$m timeout 300 python bench.py --skip-cpu --e2e-steps 0 --no-stages > gpurun_out/bench14_c2_pdl$m.log 2>&1; done
for m in 11 31; do UP_PDL_MASK=$m timeout 400 python bench.py --skip-cpu --config c5 --e2e-steps 0 > gpurun_out/bench14_c5_pdl$m.log 2>&1; done
timeout 300 python bench.py --skip-cpu --config c1 --e2e-steps 0 > gpurun_out/bench14_c1.log 2>&1
