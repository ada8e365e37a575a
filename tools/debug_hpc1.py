"""Dev (GPU box): HPC=1 (MHA) scorer vs oracle over shapes, to localise a mismatch."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, paper_2605_06221_b200 as up
from paper_2605_06221_b200.synthetic import make_batch
port = oracle.port()
for Hq, D, lengths, n, G in [(4, 128, [128], 128, 64), (4, 128, [256], 128, 64), (4, 128, [777], 128, 64),
                             (4, 128, [777], 64, 64), (4, 128, [2048], 128, 64), (1, 128, [777], 128, 64),
                             (4, 256, [777], 128, 64), (8, 128, [4096], 128, 64), (4, 128, [777], 128, 32)]:
    cfg = dict(query_window_n=n, block_size_g=G, sink_count_a=128, top_p=0.99)
    sb = make_batch(lengths, Hq, Hq, D, 64, regime="planted", block_size_g=G, seed=sum(lengths) + D)
    res = up.score_blocks_varlen(sb.q, sb.k, sb.cu_seqlens, up.ScoreConfig(**cfg), up.HeadLayout(Hq, Hq, D), check=True)
    bs = res.block_scores.cpu().numpy().astype(np.float64)
    e = lengths[0]
    _, want, _ = port.score_tokens(sb.q[:e].float().reshape(e, -1).cpu().numpy(), sb.k[:e].float().reshape(e, -1).cpu().numpy(), Hq, Hq, **cfg)
    got = bs[:len(want)]
    rel = np.abs(got - want) / np.maximum(np.abs(want), 1e-30)
    print(f"Hq={Hq} D={D} N={lengths} n={n} G={G}: worst rel {rel.max():.2e}  first bad {np.flatnonzero(rel > 1e-3)[:8]}  ratio {np.round(got[:6] / want[:6], 3)}")
