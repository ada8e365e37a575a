"""Dev (GPU box): which select path breaks stream capture?  argv[1] = lengths (comma list)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_06221_b200 as up
lengths = [int(x) for x in sys.argv[1].split(",")]
G = 64
nbs = [(n + G - 1) // G for n in lengths]
rng = np.random.default_rng(1)
scores = torch.from_numpy((rng.random(sum(nbs)) ** 7).astype(np.float32)).cuda()
cu = torch.tensor(np.concatenate([[0], np.cumsum(lengths)]), dtype=torch.int32, device="cuda")
cub = torch.tensor(np.concatenate([[0], np.cumsum(nbs)]), dtype=torch.int32, device="cuda")
cfg = up.ScoreConfig()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    sel = up.select_varlen(scores, cub, cu, cfg)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    try:
        with torch.cuda.graph(g, stream=s):
            up.select_varlen(scores, cub, cu, cfg, out=sel)
        g.replay(); torch.cuda.synchronize()
        print("OK", lengths, os.environ.get("UP_SELECT_FORK"))
    except Exception as e:
        print("FAIL", lengths, os.environ.get("UP_SELECT_FORK"), str(e).splitlines()[0])
