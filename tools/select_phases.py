"""Dev (GPU box): clock64 stamps of select CTA 0's phases (UP_SELECT_DEBUG=1) for small
requests -- start, before the crossing search, after it, after the decisions, after the
per-request epilogue (finish_request + fused expansion)."""
import ctypes, os, sys
os.environ["UP_SELECT_DEBUG"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_06221_b200 as up
for N in (4096, 32768):
    G = 64
    nb = (N + G - 1) // G
    rng = np.random.default_rng(0)
    s = rng.random(nb).astype(np.float32) ** 8
    s[rng.random(nb) < 0.25] += 0.5  # planted-like: a quarter of the blocks hot
    scores = torch.from_numpy(s).cuda()
    cu = torch.tensor([0, N], dtype=torch.int32, device="cuda")
    cub = torch.tensor([0, nb], dtype=torch.int32, device="cuda")
    out = None
    for _ in range(5):
        out = up.select_varlen(scores, cub, cu, up.ScoreConfig(), max_tokens=N, out=out)
    torch.cuda.synchronize()
    h = (ctypes.c_ulonglong * 16)()
    up.lib.up_internal_select_debug(h)
    st = sorted([(i, h[i]) for i in range(9) if h[i]], key=lambda x: x[1])
    print(f"N={N}: " + " ".join(f"{a}->{b}:{tb - ta}" for (a, ta), (b, tb) in zip(st, st[1:])), "cycles")
