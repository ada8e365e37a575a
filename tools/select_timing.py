import os, sys, torch, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_06221_b200 as up
def run(lengths, p, reps=20):
    G = 64
    nbs = [(n + G - 1)//G for n in lengths]
    rng = np.random.default_rng(0)
    scores = torch.from_numpy((rng.random(sum(nbs)) ** 8).astype(np.float32)).cuda()
    cu = torch.tensor(np.concatenate([[0], np.cumsum(lengths)]), dtype=torch.int32, device="cuda")
    cub = torch.tensor(np.concatenate([[0], np.cumsum(nbs)]), dtype=torch.int32, device="cuda")
    cfg = up.ScoreConfig(top_p=p)
    T = int(cu[-1])
    out = up.select_varlen(scores, cub, cu, cfg, check=True, max_tokens=T)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        up.select_varlen(scores, cub, cu, cfg, out=out, max_tokens=T)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps): up.select_varlen(scores, cub, cu, cfg, out=out, max_tokens=T)
        g.replay(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); g.replay(); e1.record(s)
    torch.cuda.synchronize()
    print(f"lengths={lengths[:2]}x{len(lengths)} p={p}: {e0.elapsed_time(e1)/reps*1000:.1f} us per launch (graph)")
run([32768]*4, 0.99)
run([32768]*4, 1.0)
run([4096], 0.99)
run([131072], 0.99)
run([128]*4, 0.99)
run([32768]*64, 0.99)
if os.environ.get("UP_SELECT_DEBUG"):
    import ctypes
    for lengths, p in (([32768]*4, 0.99), ([131072], 0.99), ([32768]*4, 1.0)):
        G=64; nbs=[(n+G-1)//G for n in lengths]
        rng=np.random.default_rng(0)
        scores=torch.from_numpy((rng.random(sum(nbs))**8).astype(np.float32)).cuda()
        cu=torch.tensor(np.concatenate([[0],np.cumsum(lengths)]),dtype=torch.int32,device="cuda")
        cub=torch.tensor(np.concatenate([[0],np.cumsum(nbs)]),dtype=torch.int32,device="cuda")
        up.select_varlen(scores,cub,cu,up.ScoreConfig(top_p=p),check=True)
        buf=np.zeros(16,np.uint64)
        up.lib.up_internal_select_debug(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_ulonglong)))
        b=buf.astype(np.int64); print(lengths[0], p, "phase cycles:", np.diff(b[:6]).tolist())
from paper_2605_06221_b200.synthetic import loguniform_lengths
run(loguniform_lengths(64, 4096, 131072, 5), 0.99)
