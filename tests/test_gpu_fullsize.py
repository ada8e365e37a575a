"""GPU parity at the BASELINE.json configuration sizes, through size-independent properties
and an fp64 PyTorch restatement of the scorer (too large for the CPU oracle in test time):

* block scores vs an fp64 dense softmax of the same bf16 inputs (importance.cpp:17-90
  restated with torch.float64): rtol 1e-3;
* mass conservation: Σ_g b_g·|g| = #q-heads per request (each head's softmax rows sum to 1,
  averaged over n_eff rows; test_importance.cpp:111-126);
* keep masks bit-exact vs the reference's top_p_select (oracle port) on the GPU's block
  scores, for every request;
* compaction byte-exact vs torch gathers; cu_seqlens_out = per-segment kept counts;
* reconstitution round trip restores the pre-drop buffer exactly.
"""
import numpy as np
import pytest
import torch

from paper_2605_06221_b200.synthetic import MODEL_SHAPES, make_batch

pytestmark = pytest.mark.gpu

CFG = dict(query_window_n=128, block_size_g=64, sink_count_a=128, top_p=0.99)


def _fp64_block_scores(q, k, s, e, Hq, Hkv, n, G):
    """importance.cpp:17-90 in float64 on the device: last-n queries vs all keys, causal
    mask in the tail, softmax over keys, mean over rows, sum over heads, mean per block."""
    N = e - s
    neff = min(n, N)
    D = q.shape[2]
    grp = Hq // Hkv
    qt = q[e - neff:e].to(torch.float64)            # [neff, Hq, D]
    kk = k[s:e].to(torch.float64)                   # [N, Hkv, D]
    tok = torch.zeros(N, dtype=torch.float64, device=q.device)
    rows = torch.arange(neff, device=q.device)
    cols = torch.arange(N, device=q.device)
    mask = cols[None, :] > (N - neff + rows)[:, None]
    for h in range(Hq):
        sc = qt[:, h, :] @ kk[:, h // grp, :].T / np.sqrt(D)
        sc.masked_fill_(mask, float("-inf"))
        tok += torch.softmax(sc, dim=1).sum(0) / neff
    nb = (N + G - 1) // G
    pad = torch.zeros(nb * G, dtype=torch.float64, device=q.device)
    pad[:N] = tok
    sizes = torch.full((nb,), G, dtype=torch.float64, device=q.device)
    sizes[-1] = N - (nb - 1) * G
    return pad.view(nb, G).sum(1) / sizes


def _check_layer(up, port, sb, Hq, Hkv, D, lengths, cfg, tp=1, exact_requests=(0,)):
    sc = up.ScoreConfig(**cfg)
    heads = up.HeadLayout(Hq, Hkv, D)
    if tp > 1:
        res = up.score_blocks_tp(sb.q, sb.k, sb.cu_seqlens, sc, tp, heads, check=True)
    else:
        res = up.score_blocks_varlen(sb.q, sb.k, sb.cu_seqlens, sc, heads, check=True)
    cu = sb.cu_seqlens.cpu().numpy()
    cub = res.cu_blocks.cpu().numpy()
    bs = res.block_scores[:int(cub[-1])].double()
    G = cfg["block_size_g"]
    for r in range(len(lengths)):
        s, e = int(cu[r]), int(cu[r + 1])
        b = bs[cub[r]:cub[r + 1]]
        sizes = torch.full_like(b, G)
        sizes[-1] = (e - s) - (b.numel() - 1) * G
        mass = float((b * sizes).sum())
        assert abs(mass - Hq) < 1e-3 * Hq, (r, mass)
        if r in exact_requests:
            want = _fp64_block_scores(sb.q, sb.k, s, e, Hq, Hkv, cfg["query_window_n"], G)
            err = (b - want).abs()
            atol = 1e-6 * float(want.sum()) / want.numel()
            bad = err > 1e-3 * want.abs() + atol
            assert not bool(bad.any()), f"request {r}: {int(bad.sum())} blocks off, worst {float((err / want).max()):.2e}"
            print(f"request {r}: N={e - s} mass={mass:.6f} worst rel err {float((err / want).max()):.2e}")
    # selection: bit-exact vs the reference top_p_select on the GPU's own block scores
    sel = up.select_varlen(res.block_scores, res.cu_blocks, sb.cu_seqlens, sc, check=True)
    keep = sel.keep.cpu().numpy()
    bsh = res.block_scores.cpu().numpy()
    kstar = sel.cutoff_rank.cpu().numpy()
    for r in range(len(lengths)):
        s, e = int(cu[r]), int(cu[r + 1])
        want = port.top_p_select(bsh[cub[r]:cub[r + 1]], e - s, **cfg)
        assert np.array_equal(keep[s:e], want.keep_mask), f"keep mask of request {r}"
        assert int(kstar[r]) == want.cutoff_rank
    # compaction: byte-exact gathers, new cu_seqlens, then the reconstitution round trip
    planes = [sb.hidden, sb.k, sb.v, sb.positions]
    out = up.compact_varlen(sel.keep, sb.cu_seqlens, planes, check=True)
    n = int(out.num_out.item())
    idx = out.retained_index[:n].long()
    assert bool((idx[1:] > idx[:-1]).all())
    for src, dst in zip(planes, out.planes):
        assert torch.equal(dst[:n], src[idx])
    kept = [int(keep[int(cu[r]):int(cu[r + 1])].sum()) for r in range(len(lengths))]
    assert out.cu_seqlens.cpu().tolist() == np.concatenate([[0], np.cumsum(kept)]).tolist()
    pre = sb.hidden.clone()
    pre[idx] = 0  # wipe the retained rows; the unwind must restore them exactly
    up.reconstitute_varlen([out.planes[0]], out, [pre])
    assert torch.equal(pre, sb.hidden)
    return n / sum(lengths)


def test_llama_4x32k_full_layer(up, port):
    """BASELINE config 2 layer (LLaMA-3.1-8B shape, 4 x 32K)."""
    shp = MODEL_SHAPES["llama3.1-8b"]
    lengths = [32768] * 4
    sb = make_batch(lengths, shp["num_q_heads"], shp["num_kv_heads"], shp["head_dim"], shp["hidden"],
                    regime="planted", seed=11)
    rho = _check_layer(up, port, sb, shp["num_q_heads"], shp["num_kv_heads"], shp["head_dim"], lengths, CFG,
                       exact_requests=(0, 3))
    assert 0.1 < rho < 0.6


def test_qwen3_next_128k_tp8_full_layer(up, port):
    """BASELINE config 3 layer (Qwen3-Next full-attention shape, 1 x 128K, TP=8 shards)."""
    shp = MODEL_SHAPES["qwen3-next-80b-a3b"]
    lengths = [131072]
    sb = make_batch(lengths, shp["num_q_heads"], shp["num_kv_heads"], shp["head_dim"], shp["hidden"],
                    regime="planted", seed=12)
    _check_layer(up, port, sb, shp["num_q_heads"], shp["num_kv_heads"], shp["head_dim"], lengths, CFG, tp=8)


def test_gemma3_varlen_64k_layer(up, port):
    """BASELINE config 4 shape (Gemma-3-12B, p = 0.98), four 64K requests."""
    shp = MODEL_SHAPES["gemma3-12b"]
    lengths = [65536] * 4
    cfg = dict(CFG, top_p=0.98)
    sb = make_batch(lengths, shp["num_q_heads"], shp["num_kv_heads"], shp["head_dim"], shp["hidden"],
                    regime="planted", seed=13)
    _check_layer(up, port, sb, shp["num_q_heads"], shp["num_kv_heads"], shp["head_dim"], lengths, cfg,
                 exact_requests=(1,))


def test_mixed_stream_64_requests(up, port):
    """BASELINE config 5 stream (64 requests, 4K-128K log-uniform): per-request checks."""
    from paper_2605_06221_b200.synthetic import loguniform_lengths
    shp = MODEL_SHAPES["llama3.1-8b"]
    lengths = loguniform_lengths(64, 4096, 131072, 5)
    sb = make_batch(lengths, shp["num_q_heads"], shp["num_kv_heads"], shp["head_dim"], shp["hidden"],
                    regime="planted", seed=14)
    _check_layer(up, port, sb, shp["num_q_heads"], shp["num_kv_heads"], shp["head_dim"], lengths, CFG,
                 exact_requests=(0, 31))


def test_one_million_token_request_tp_rank(up, port):
    """Maximum request size: a 2^20-token (1M context) request at one Qwen3-Next TP=8 rank's
    head slice (2 q-heads, 1 kv-head, D = 256) -- 16384 blocks, the most the on-chip select
    sort holds -- through score (fp64 restatement), select (bit-exact), compaction and the
    reconstitution round trip."""
    lengths = [1 << 20]
    sb = make_batch(lengths, 2, 1, 256, 512, regime="planted", seed=15)
    rho = _check_layer(up, port, sb, 2, 1, 256, lengths, CFG)
    assert 0.05 < rho < 0.8
