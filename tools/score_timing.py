"""Dev timing of the scorer stage (scorer + pair weights + combine) in a CUDA graph.
SHAPE=llama|gemma|qwen|qwen-tp8 (default llama: 4x32K), REGIME=planted|iid."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_06221_b200 as up
from paper_2605_06221_b200.synthetic import make_batch

SHAPES = {  # Hq, Hkv, D, lengths, tp
    "llama": (32, 8, 128, [32768] * 4, 1),
    "llama4k": (32, 8, 128, [4096], 1),
    "gemma": (16, 8, 256, [65536] * 4, 1),
    "qwen": (16, 2, 256, [131072], 1),
    "qwen-tp8": (16, 2, 256, [131072], 8),
    "mha": (32, 32, 128, [32768] * 4, 1),
    "mha256": (16, 16, 256, [65536] * 2, 1),
    "gqa2": (32, 16, 128, [32768] * 4, 1),
    "mixed": (32, 32, 128, [100] * 2000 + [65536], 1),
    "mixed-llama": (32, 8, 128, [100] * 2000 + [65536], 1),
    "short-mha": (32, 32, 128, [100] * 2000, 1),
}
Hq, Hkv, D, L, tp = SHAPES[os.environ.get("SHAPE", "llama")]
sb = make_batch(L, Hq, Hkv, D, 64, regime=os.environ.get("REGIME", "planted"), seed=1, device="cuda", with_v=False)
cfg = up.ScoreConfig(block_size_g=int(os.environ.get("G", "64")), query_window_n=int(os.environ.get("NQ", "128"))); h = up.HeadLayout(Hq, Hkv, D)
run = (lambda: up.score_blocks_tp(sb.q, sb.k, sb.cu_seqlens, cfg, tp, h, out=out)) if tp > 1 else \
      (lambda: up.score_blocks_varlen(sb.q, sb.k, sb.cu_seqlens, cfg, h, out=out))
out = None
out = run()
torch.cuda.synchronize()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    run(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(10): run()
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s); g.replay(); e1.record(s)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
flops = sum(2 * min(cfg.query_window_n, n) * n * D * Hq for n in L)
print(f"{os.environ.get('SHAPE', 'llama')}: {ms:.4f} ms  {flops / ms / 1e9:.1f} TFLOP/s")
