import os, sys, torch, ctypes, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_06221_b200 as up
from paper_2605_06221_b200.synthetic import make_batch
sb = make_batch([32768]*4, 32, 8, 128, 64, regime=os.environ.get("REGIME","planted"), seed=1, device="cuda", with_v=False)
cfg = up.ScoreConfig(); h = up.HeadLayout(32, 8, 128)
out = up.score_blocks_varlen(sb.q, sb.k, sb.cu_seqlens, cfg, h, check=not os.environ.get("NOCHECK"))
for _ in range(3): up.score_blocks_varlen(sb.q, sb.k, sb.cu_seqlens, cfg, h, out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): up.score_blocks_varlen(sb.q, sb.k, sb.cu_seqlens, cfg, h, out=out)
e1.record(); torch.cuda.synchronize()
print(os.environ.get("UP_SCORE_GRID"), os.environ.get("REGIME"), "ms", e0.elapsed_time(e1)/20)
if os.environ.get("UP_SCORE_DEBUG"):
    g = int(os.environ.get("UP_SCORE_GRID", "148"))
    buf = np.zeros(4*g, np.uint64)
    up.lib.up_internal_score_debug(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_ulonglong)), g)
    b = buf.reshape(g, 4).astype(np.int64)
    t0 = b[:,0].min(); st = (b[:,0]-t0)/1e3; en = (b[:,1]-t0)/1e3
    order = np.argsort(-en)
    print("start us: min %.1f max %.1f; end us: min %.1f med %.1f max %.1f" % (st.min(), st.max(), en.min(), np.median(en), en.max()))
    for i in order[:8]: print(" cta", i, "sm", b[i,3], "units", b[i,2], "start %.1f end %.1f" % (st[i], en[i]))
    for i in order[-3:]: print(" cta", i, "sm", b[i,3], "units", b[i,2], "start %.1f end %.1f" % (st[i], en[i]))
