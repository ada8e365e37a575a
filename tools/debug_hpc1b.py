import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, paper_2605_06221_b200 as up
from paper_2605_06221_b200.synthetic import make_batch
port = oracle.port()
for Hq, D, lengths, n, G in [(1, 128, [384], 128, 64), (1, 128, [512], 128, 64), (1, 128, [1024], 128, 64), (1, 128, [1024], 32, 64)]:
    cfg = dict(query_window_n=n, block_size_g=G, sink_count_a=128, top_p=0.99)
    sb = make_batch(lengths, Hq, Hq, D, 64, regime=os.environ.get("REGIME", "planted"), block_size_g=G, seed=3)
    res = up.score_blocks_varlen(sb.q, sb.k, sb.cu_seqlens, up.ScoreConfig(**cfg), up.HeadLayout(Hq, Hq, D), check=True)
    bs = res.block_scores.cpu().numpy().astype(np.float64)
    e = lengths[0]
    _, want, _ = port.score_tokens(sb.q[:e].float().reshape(e, -1).cpu().numpy(), sb.k[:e].float().reshape(e, -1).cpu().numpy(), Hq, Hq, **cfg)
    got = bs[:len(want)]
    print(f"Hq={Hq} N={lengths} n={n}: ratios {np.round(got / want, 3).tolist()}")
