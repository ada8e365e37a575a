import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2605_06221_b200 as up, oracle
from paper_2605_06221_b200.synthetic import make_batch
for L in ([1000], [4096], [300, 700]):
    sb = make_batch(L, 4, 1, 128, 64, regime="iid", seed=3, device="cuda")
    cfg = up.ScoreConfig()
    out = up.score_blocks_varlen(sb.q, sb.k, sb.cu_seqlens, cfg, up.HeadLayout(4, 1, 128), check=True)
    torch.cuda.synchronize()
    cu = sb.cu_seqlens.cpu().numpy(); cub = out.cu_blocks.cpu().numpy(); bs = out.block_scores.cpu().numpy()
    port = oracle.port()
    for r in range(len(L)):
        s, e = cu[r], cu[r+1]
        q = sb.q[s:e].float().reshape(e-s, -1).cpu().numpy(); k = sb.k[s:e].float().reshape(e-s, -1).cpu().numpy()
        _, want, _ = port.score_tokens(q, k, 4, 1, query_window_n=128, block_size_g=64, sink_count_a=128, top_p=0.99)
        got = bs[cub[r]:cub[r+1]]
        print(os.environ.get("UP_SCORE_GRID"), L, r, "ratio", np.round(got / want, 3)[:12], "sum got", got.sum(), "want", want.sum())
