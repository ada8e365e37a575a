"""Dev (GPU box): per-CTA globaltimer spans of the tensor-core scorer (UP_SCORE_DEBUG=1) for
a small launch (LLaMA 1x4K by default) -- when CTAs start, how long each runs."""
import ctypes, os, sys
os.environ["UP_SCORE_DEBUG"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_06221_b200 as up
from paper_2605_06221_b200.synthetic import make_batch
L = [int(x) for x in os.environ.get("LENGTHS", "4096").split(",")]
sb = make_batch(L, 32, 8, 128, 64, regime="planted", seed=1, device="cuda", with_v=False)
cfg, h = up.ScoreConfig(), up.HeadLayout(32, 8, 128)
out = None
for _ in range(5):
    out = up.score_blocks_varlen(sb.q, sb.k, sb.cu_seqlens, cfg, h, out=out)
torch.cuda.synchronize()
n = 148
buf = (ctypes.c_ulonglong * (4 * n))()
up.lib.up_internal_score_debug(buf, n)
rec = [(buf[4 * i], buf[4 * i + 1], buf[4 * i + 2]) for i in range(n)]
t0 = min(r[0] for r in rec)
starts = sorted((r[0] - t0) / 1e3 for r in rec)
durs = sorted((r[1] - r[0]) / 1e3 for r in rec)
ends = sorted((r[1] - t0) / 1e3 for r in rec)
units = sorted(r[2] for r in rec)
print(f"lengths={L}: start spread {starts[0]:.2f}..{starts[-1]:.2f} us; CTA span min/med/max "
      f"{durs[0]:.2f}/{durs[len(durs)//2]:.2f}/{durs[-1]:.2f} us; last end {ends[-1]:.2f} us; units/CTA {units[0]}..{units[-1]}")
ph = (ctypes.c_ulonglong * (4 * n))()
if up.lib.up_internal_score_phases(ph, n) == 0:
    for k, name in enumerate(["Q landed (MMA warp)", "first S region (epilogue)", "first item done"]):
        d = sorted((ph[4 * i + k] - rec[i][0]) / 1e3 for i in range(n) if ph[4 * i + k])
        if d:
            print(f"  {name}: min/med/max {d[0]:.2f}/{d[len(d)//2]:.2f}/{d[-1]:.2f} us after CTA start")
