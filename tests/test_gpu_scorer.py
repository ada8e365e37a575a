"""GPU parity: block-wise importance scorer vs the CPU oracle (importance.cpp:17-132).

Tolerance (north star): block scores within rtol 1e-3 of the oracle on identical bf16
inputs (GPU: bf16 in / fp32 accumulate; oracle: the same values upcast to fp32, double
accumulation), plus an absolute floor of 1e-6 x the block-score mass for blocks whose
score underflows fp32 relative to its row maxima.
"""
import numpy as np
import pytest
import torch

from paper_2605_06221_b200.synthetic import make_batch

pytestmark = pytest.mark.gpu

RTOL = 1e-3


def _oracle_blocks(port, sb, r, Hq, Hkv, cfg):
    cu = sb.cu_seqlens.cpu().numpy()
    s, e = int(cu[r]), int(cu[r + 1])
    q = sb.q[s:e].float().reshape(e - s, -1).cpu().numpy()
    k = sb.k[s:e].float().reshape(e - s, -1).cpu().numpy()
    tok, blk, _ = port.score_tokens(q, k, Hq, Hkv, **cfg)
    return tok, blk


def _assert_blocks_close(got, want):
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    atol = 1e-6 * max(want.sum(), 1e-30) / max(len(want), 1)
    err = np.abs(got - want)
    bad = err > RTOL * np.abs(want) + atol
    assert not bad.any(), (f"{bad.sum()} / {len(want)} blocks off; worst rel "
                           f"{(err / np.maximum(np.abs(want), 1e-30)).max():.3e}")


@pytest.mark.parametrize("Hq,Hkv,D,lengths,n,G", [
    (8, 2, 128, [1000], 128, 64),          # GQA 4 -> HPC 4 (LLaMA-like)
    (8, 2, 128, [700, 129, 64, 2000], 128, 64),  # varlen, short segments
    (4, 1, 128, [300, 1], 128, 64),        # single-token segment
    (8, 1, 64, [1500], 128, 64),           # D=64, HPC 8
    (4, 2, 256, [900, 333], 128, 64),      # D=256 (Gemma / Qwen head dim)
    (4, 4, 128, [777], 128, 64),           # MHA, HPC 1 (score_tcw TS, four parity warpgroups)
    (8, 8, 128, [2000, 64, 900], 128, 32), # MHA varlen, G=32
    (4, 4, 256, [1500, 300], 128, 64),     # MHA at D=256
    (16, 8, 256, [3000, 700], 128, 128),   # Gemma-3 layout at G=128 (score_tc: D=256 leaves too few TMEM regions)
    (4, 4, 128, [1500, 90], 128, 128),     # MHA at G=128 (HPC 1, paired-subtile parity units)
    (8, 2, 128, [2048, 300], 32, 128),     # packed rows (P = 4, HPC 1) at G=128
    (16, 4, 128, [2500, 128, 900], 128, 128),  # GQA 4 at G=128 (HPC 2, D=128)
    # many one-unit items ahead of long ones (~15 items per CTA): a parity warpgroup of the
    # CTA at the boundary sees a run of items that never reach its parity, then a long item
    # (TMEM ring phases, HPC 1)
    (8, 8, 128, [100] * 200 + [6000, 700], 128, 64),
    (4, 4, 256, [90] * 300 + [4000], 128, 32),
    (8, 8, 128, [120] * 200 + [6000], 128, 128),
    # the D <= 128 parity variants walk only their own subtiles (stride NPAR, pairs at
    # G = 128): GQA-2 and D = 64 with short items ahead of long ones, every G
    (16, 8, 128, [90] * 150 + [3000, 257], 128, 32),
    (16, 8, 128, [130] * 120 + [4000], 128, 128),
    (8, 4, 64, [100] * 100 + [2500], 128, 128),
    (8, 4, 64, [700, 64, 1900], 128, 64),
    (8, 2, 128, [1024, 513], 64, 32),      # n=64, G=32
    (8, 2, 128, [2048], 128, 128),         # G=128
    (8, 2, 128, [1300], 100, 96),          # n < 128, G not a power of two
    (4, 2, 256, [700, 1200], 128, 32),     # D=256, G=32 (two warpgroups per head, 2 blocks/subtile)
    (2, 1, 256, [5000], 128, 64),          # Qwen3-Next TP-rank slice: 2 q-heads on 1 kv-head
    (4, 2, 256, [1000], 128, 128),         # D=256, G=128 -> two-warpgroup kernel, HPC 1
    (8, 4, 128, [1500, 260], 128, 64),     # GQA 2 at D=128 (HPC 2, parity warpgroups)
    (8, 2, 64, [900], 128, 64),            # D=64, HPC 4
    (4, 2, 64, [650], 128, 32),            # D=64, HPC 2
    (16, 8, 256, [3000, 64, 4100], 128, 64),  # Gemma-3 layout, varlen
])
def test_tc_scorer_matches_oracle(up, port, Hq, Hkv, D, lengths, n, G):
    cfg = dict(query_window_n=n, block_size_g=G, sink_count_a=128, top_p=0.99)
    sb = make_batch(lengths, Hq, Hkv, D, 64, regime="planted", block_size_g=G, seed=sum(lengths) + D)
    sc = up.ScoreConfig(**cfg)
    heads = up.HeadLayout(Hq, Hkv, D)
    import paper_2605_06221_b200._capi as capi
    import ctypes
    assert up.lib.up_scorer_kind(ctypes.byref(heads.c(Hq * D, Hkv * D)), ctypes.byref(sc.c()), 0) == 1
    res = up.score_blocks_varlen(sb.q, sb.k, sb.cu_seqlens, sc, heads, check=True)
    cub = res.cu_blocks.cpu().numpy()
    bs = res.block_scores.cpu().numpy()
    for r in range(len(lengths)):
        _, want = _oracle_blocks(port, sb, r, Hq, Hkv, cfg)
        got = bs[cub[r]:cub[r + 1]]
        assert len(got) == len(want)
        _assert_blocks_close(got, want)


@pytest.mark.parametrize("Hq,Hkv,D,lengths,n,G", [
    (8, 8, 8, [40], 16, 8),              # score_default.json fixture shape (n=16, G=8)
    (4, 2, 32, [300, 17, 5], 8, 4),
    (2, 1, 64, [130], 200, 10),          # n > N (clamped), odd G
])
def test_simt_scorer_matches_oracle_tokens_and_blocks(up, port, Hq, Hkv, D, lengths, n, G):
    cfg = dict(query_window_n=n, block_size_g=G, sink_count_a=8, top_p=0.9)
    sb = make_batch(lengths, Hq, Hkv, D, 16, regime="iid", seed=7)
    res = up.score_blocks_varlen(sb.q, sb.k, sb.cu_seqlens, up.ScoreConfig(**cfg),
                                 up.HeadLayout(Hq, Hkv, D), want_token_scores=True, check=True)
    cub = res.cu_blocks.cpu().numpy()
    cu = sb.cu_seqlens.cpu().numpy()
    for r in range(len(lengths)):
        tok, blk = _oracle_blocks(port, sb, r, Hq, Hkv, cfg)
        got_t = res.token_scores[cu[r]:cu[r + 1]].cpu().numpy()
        np.testing.assert_allclose(got_t, tok, rtol=RTOL, atol=1e-7)
        _assert_blocks_close(res.block_scores[cub[r]:cub[r + 1]].cpu().numpy(), blk)
        # mass conservation: token scores of one request sum to #heads (test_importance.cpp:111-126)
        assert abs(got_t.sum() - Hq) < 1e-3 * Hq


def test_tc_and_simt_agree(up):
    sb = make_batch([1200, 300], 8, 2, 128, 64, regime="planted", seed=3)
    sc = up.ScoreConfig()
    h = up.HeadLayout(8, 2, 128)
    a = up.score_blocks_varlen(sb.q, sb.k, sb.cu_seqlens, sc, h, check=True)
    b = up.score_blocks_varlen(sb.q, sb.k, sb.cu_seqlens, sc, h, want_token_scores=True, check=True)
    nb = int(a.cu_blocks[-1].item())
    _assert_blocks_close(a.block_scores[:nb].cpu().numpy(), b.block_scores[:nb].cpu().numpy())


def test_drop_disabled_segments_are_skipped(up, port):
    sb = make_batch([500, 1, 800], 8, 2, 128, 64, regime="planted", seed=11)
    en = torch.tensor([1, 0, 1], dtype=torch.uint8, device="cuda")
    res = up.score_blocks_varlen(sb.q, sb.k, sb.cu_seqlens, up.ScoreConfig(), up.HeadLayout(8, 2, 128),
                                 drop_enabled=en, check=True)
    cub = res.cu_blocks.cpu().numpy()
    assert list(cub) == [0, 8, 9, 22]
    assert float(res.block_scores[8].item()) == 0.0
    for r in (0, 2):
        _, want = _oracle_blocks(port, sb, r, 8, 2, dict(query_window_n=128, block_size_g=64,
                                                         sink_count_a=128, top_p=0.99))
        _assert_blocks_close(res.block_scores[cub[r]:cub[r + 1]].cpu().numpy(), want)


def test_score_tokens_mirror_head_ranges_and_tp_sum(up, port):
    """score_tokens_heads + allreduce over shards == unsharded (test_tp_sim.cpp:45-58)."""
    N, H, Hkv, D = 600, 8, 2, 128
    g = torch.Generator().manual_seed(5)
    q = torch.randn(N, H * D, generator=g).to(torch.bfloat16).cuda()
    k = torch.randn(N, Hkv * D, generator=g).to(torch.bfloat16).cuda()
    cfg = up.ScoreConfig(query_window_n=128, block_size_g=64, sink_count_a=16, top_p=0.9)
    full = up.score_tokens(q, k, H, cfg, num_kv_heads=Hkv, want_token_scores=False)
    for tp in (1, 2, 4, 8):
        shards = up.sharded_block_scores(q, k, H, cfg, tp, num_kv_heads=Hkv)
        red = up.allreduce_scores(shards).cpu().numpy()
        _assert_blocks_close(red, full.block_scores.cpu().numpy())
    with pytest.raises(up.ConfigError):
        up.sharded_block_scores(q, k, H, cfg, 3, num_kv_heads=Hkv)


@pytest.mark.parametrize("Hq,Hkv,D,tp,lengths", [
    (16, 2, 256, 8, [3000]),      # Qwen3-Next full-attention layer at TP=8 (2 heads per shard)
    (32, 8, 128, 8, [1100, 700]),  # LLaMA layout at TP=8 (4 heads per shard)
    (8, 2, 128, 2, [900]),
    (4, 4, 32, 4, [300]),         # generic shape (SIMT shards + ordered reduce kernel)
])
def test_score_blocks_tp_matches_reference_sharding(up, port, ref, Hq, Hkv, D, tp, lengths):
    """up_score_blocks_tp == sharded_block_scores + allreduce_scores (tp_sim.cpp:12-49):
    every shard within rtol of the reference shard, the reduction bitwise equal to the
    ascending-shard fp32 sum of the returned shard partials."""
    cfg = dict(query_window_n=128, block_size_g=64, sink_count_a=128, top_p=0.99)
    sb = make_batch(lengths, Hq, Hkv, D, 64, regime="planted", seed=len(lengths) * 31 + D)
    res = up.score_blocks_tp(sb.q, sb.k, sb.cu_seqlens, up.ScoreConfig(**cfg), tp, up.HeadLayout(Hq, Hkv, D),
                             check=True)
    cub = res.cu_blocks.cpu().numpy()
    cu = sb.cu_seqlens.cpu().numpy()
    shards = res.shard_scores.cpu().numpy()
    red = res.block_scores.cpu().numpy()
    nb = int(cub[-1])
    want_red = np.zeros(nb, np.float32)
    for t in range(tp):
        want_red = (want_red + shards[t, :nb]).astype(np.float32)
    assert np.array_equal(red[:nb].view(np.uint32), want_red.view(np.uint32))
    for r in range(len(lengths)):
        s, e = int(cu[r]), int(cu[r + 1])
        q = sb.q[s:e].float().reshape(e - s, -1).cpu().numpy()
        k = sb.k[s:e].float().reshape(e - s, -1).cpu().numpy()
        ref_shards, ref_red = ref.sharded_allreduce(q, k, Hq, Hkv, tp, **cfg)
        for t in range(tp):
            _assert_blocks_close(shards[t, cub[r]:cub[r + 1]], ref_shards[t])
        _assert_blocks_close(red[cub[r]:cub[r + 1]], ref_red)


def test_score_blocks_tp_rejects_bad_degree(up):
    sb = make_batch([200], 8, 2, 128, 64, seed=1)
    for tp in (0, 3):
        with pytest.raises(up.ConfigError):
            up.score_blocks_tp(sb.q, sb.k, sb.cu_seqlens, up.ScoreConfig(), tp, up.HeadLayout(8, 2, 128))


@pytest.mark.parametrize("R,maxlen", [(300, 400), (4100, 40)])
def test_many_requests(up, port, R, maxlen):
    """Continuous batches with many segments: up to 4096 (kTcwMaxRequests) score_tcw plans
    them in shared memory; beyond, the two-warpgroup kernel or, when its plan does not fit
    either, the SIMT scorer serves the batch.  Every sampled segment matches the oracle."""
    rng = np.random.default_rng(8)
    lengths = [int(x) for x in rng.integers(1, maxlen, size=R)]
    cfg = dict(query_window_n=128, block_size_g=64, sink_count_a=128, top_p=0.99)
    sb = make_batch(lengths, 8, 2, 128, 16, regime="planted", seed=8)
    res = up.score_blocks_varlen(sb.q, sb.k, sb.cu_seqlens, up.ScoreConfig(**cfg), up.HeadLayout(8, 2, 128),
                                 check=True)
    cub = res.cu_blocks.cpu().numpy()
    bs = res.block_scores.cpu().numpy()
    for r in range(0, len(lengths), 37):
        _, want = _oracle_blocks(port, sb, r, 8, 2, cfg)
        _assert_blocks_close(bs[cub[r]:cub[r + 1]], want)


def test_unaligned_q_takes_the_simt_path(up, port):
    """A q view whose base is not 16-byte aligned cannot feed TMA: the scorer must still
    answer (SIMT path) within rtol of the oracle."""
    lengths = [500]
    cfg = dict(query_window_n=128, block_size_g=64, sink_count_a=128, top_p=0.99)
    sb = make_batch(lengths, 4, 1, 128, 16, regime="planted", seed=5)
    buf = torch.empty(sb.q.numel() + 1, dtype=torch.bfloat16, device="cuda")
    q = buf[1:].view(sb.q.shape)
    q.copy_(sb.q)
    assert q.data_ptr() % 16 != 0
    res = up.score_blocks_varlen(q, sb.k, sb.cu_seqlens, up.ScoreConfig(**cfg), up.HeadLayout(4, 1, 128), check=True)
    _, want = _oracle_blocks(port, sb, 0, 4, 1, cfg)
    _assert_blocks_close(res.block_scores[:len(want)].cpu().numpy(), want)


@pytest.mark.parametrize("Hq,Hkv,D,lengths", [
    (32, 8, 128, [1000, 50]),     # wide scorer, HPC 4; the last segment is shorter than n
    (16, 2, 256, [700, 90]),      # TS scorer (HPC 2, Q in TMEM)
    (4, 4, 64, [500, 33]),        # two-warpgroup scorer
])
def test_scores_ignore_garbage_past_the_batch(up, Hq, Hkv, D, lengths):
    """Capacity-sized q/k buffers whose rows past cu_seqlens[-1] hold NaN: the query-window
    tile of a short last segment and its ragged last key tile read those rows, yet the block
    scores equal the clean-buffer scores bit for bit."""
    from paper_2605_06221_b200.synthetic import make_batch
    sb = make_batch(lengths, Hq, Hkv, D, 32, regime="planted", seed=9)
    n, cap = sum(lengths), sum(lengths) + 300
    cfg = up.ScoreConfig()
    heads = up.HeadLayout(Hq, Hkv, D)
    clean = up.score_blocks_varlen(sb.q, sb.k, sb.cu_seqlens, cfg, heads, check=True)
    qp = torch.full((cap, Hq, D), float("nan"), dtype=torch.bfloat16, device="cuda")
    kp = torch.full((cap, Hkv, D), float("nan"), dtype=torch.bfloat16, device="cuda")
    qp[:n] = sb.q
    kp[:n] = sb.k
    dirty = up.score_blocks_varlen(qp, kp, sb.cu_seqlens, cfg, heads, max_tokens=cap, check=True)
    nb = int(clean.cu_blocks[-1])
    a, b = clean.block_scores[:nb], dirty.block_scores[:nb]
    assert bool(torch.isfinite(b).all())
    assert torch.equal(a, b)


_TC2_CHILD = r'''
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import oracle, paper_2605_06221_b200 as up
from paper_2605_06221_b200.synthetic import make_batch
port = oracle.port()
bad = []
for Hq, Hkv, lengths, n, G in [(8, 2, [1000], 128, 64), (8, 2, [700, 129, 64, 2000], 128, 64),
                               (8, 2, [1024, 513], 64, 32), (8, 2, [2048, 300], 128, 128), (4, 1, [300, 1], 128, 64)]:
    cfg = dict(query_window_n=n, block_size_g=G, sink_count_a=128, top_p=0.99)
    sb = make_batch(lengths, Hq, Hkv, 128, 64, regime="planted", block_size_g=G, seed=sum(lengths) + 5)
    res = up.score_blocks_varlen(sb.q, sb.k, sb.cu_seqlens, up.ScoreConfig(**cfg), up.HeadLayout(Hq, Hkv, 128), check=True)
    cu, cub, bs = sb.cu_seqlens.cpu().numpy(), res.cu_blocks.cpu().numpy(), res.block_scores.cpu().numpy().astype(np.float64)
    for r in range(len(lengths)):
        s, e = int(cu[r]), int(cu[r + 1])
        _, want, _ = port.score_tokens(sb.q[s:e].float().reshape(e - s, -1).cpu().numpy(),
                                       sb.k[s:e].float().reshape(e - s, -1).cpu().numpy(), Hq, Hkv, **cfg)
        got = bs[cub[r]:cub[r + 1]]
        atol = 1e-6 * max(want.sum(), 1e-30) / len(want)
        if len(got) != len(want) or (np.abs(got - want) > 1e-3 * np.abs(want) + atol).any():
            bad.append((Hq, Hkv, lengths, G, r))
print("TC2_BAD", bad)
'''


@pytest.mark.parametrize("env,marker", [
    ({"UP_TC2": "1"}, "pair=1"),                    # score_tc2, CTA pairs (opt-in)
    ({"UP_TCW_SPLIT": "1"}, "wide=1 hpc=4 npar=2"),  # score_tcw, SPLIT epilogue forced
    ({"UP_TCW_SPLIT": "0"}, "wide=1 hpc=4 npar=1"),  # score_tcw, one warpgroup per head forced
])
def test_scorer_variants_match_oracle(up, env, marker):
    """The GQA-4 D = 128 scorer variants, each forced in a child process (the selection is
    read once per process): score_tc2 (tcgen05.mma.cta_group::2, M = 256 over a CTA pair),
    and score_tcw with either epilogue (SPLIT: two warpgroups per head, one per 64-key half,
    each alternating between two heads; chosen automatically for small launches, see
    DESIGN.md 3(a)).  Block scores vs the oracle within rtol 1e-3 for G in {32, 64, 128},
    varlen and single-token segments."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", _TC2_CHILD, root], capture_output=True, text=True, timeout=600,
                         env=dict(os.environ, UP_SCORE_VERBOSE="1", **env))
    assert out.returncode == 0, out.stderr[-2000:]
    assert marker in out.stderr  # the variant actually ran
    assert "TC2_BAD []" in out.stdout, out.stdout[-2000:]


_TILES_CHILD = r'''
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import oracle, paper_2605_06221_b200 as up
from paper_2605_06221_b200.synthetic import make_batch
port = oracle.port()
bad = []
for Hq, Hkv, D, lengths, n, G in [(8, 2, 128, [1000, 2000, 130], 256, 64),   # Tt = 2 < HPC
                                  (32, 8, 128, [4096, 700], 512, 64),       # LLaMA heads, Tt = 4 = HPC
                                  (4, 1, 128, [1500, 90], 300, 32),         # ragged last tile
                                  (16, 2, 256, [3000, 600], 512, 64),       # Qwen3-Next heads, HPC 2 TS
                                  (8, 4, 128, [2500], 384, 128)]:           # G = 128
    cfg = dict(query_window_n=n, block_size_g=G, sink_count_a=128, top_p=0.99)
    sb = make_batch(lengths, Hq, Hkv, D, 64, regime="planted", block_size_g=G, seed=sum(lengths) + n)
    res = up.score_blocks_varlen(sb.q, sb.k, sb.cu_seqlens, up.ScoreConfig(**cfg), up.HeadLayout(Hq, Hkv, D), check=True)
    cu, cub, bs = sb.cu_seqlens.cpu().numpy(), res.cu_blocks.cpu().numpy(), res.block_scores.cpu().numpy().astype(np.float64)
    for r in range(len(lengths)):
        s, e = int(cu[r]), int(cu[r + 1])
        _, want, _ = port.score_tokens(sb.q[s:e].float().reshape(e - s, -1).cpu().numpy(),
                                       sb.k[s:e].float().reshape(e - s, -1).cpu().numpy(), Hq, Hkv, **cfg)
        got = bs[cub[r]:cub[r + 1]]
        atol = 1e-6 * max(want.sum(), 1e-30) / len(want)
        if len(got) != len(want) or (np.abs(got - want) > 1e-3 * np.abs(want) + atol).any():
            bad.append((Hq, Hkv, D, lengths, n, G, r))
print("TILES_BAD", bad)
'''


def test_query_window_beyond_128_on_tensor_cores(up):
    """n > 128 (the paper's n ablation: 32 / 128 / 512, PAPER.md Table 'last n'): the query
    window is scored as ceil(n/128) tiles of 128 rows on score_tcw (tile t of q-head h =
    virtual head h*Tt + t), not on the SIMT fallback.  Block scores vs the oracle within
    rtol 1e-3 for Tt in {2, 3, 4}, GQA 1/2/4, D 128/256, G 32/64/128, short requests."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", _TILES_CHILD, root], capture_output=True, text=True, timeout=900,
                         env=dict(os.environ, UP_SCORE_VERBOSE="1"))
    assert out.returncode == 0, out.stderr[-2000:]
    assert "wide=0" not in out.stderr and "wide=1" in out.stderr  # every call on score_tcw
    assert "TILES_BAD []" in out.stdout, out.stdout[-2000:]


@pytest.mark.parametrize("tp", [2, 4])
def test_query_tiles_tp_shards_match_reference(up, port, tp):
    """n = 256 with TP head shards (virtual heads stay contiguous per shard): the sharded
    scores' ascending-shard sum vs the oracle."""
    Hq, Hkv, D, lengths = 8, 2, 128, [1500, 700]
    cfg = dict(query_window_n=256, block_size_g=64, sink_count_a=128, top_p=0.99)
    sb = make_batch(lengths, Hq, Hkv, D, 64, regime="planted", seed=4242)
    res = up.score_blocks_tp(sb.q, sb.k, sb.cu_seqlens, up.ScoreConfig(**cfg), tp, up.HeadLayout(Hq, Hkv, D))
    cub = res.cu_blocks.cpu().numpy()
    bs = res.block_scores.cpu().numpy()
    for r in range(len(lengths)):
        _, want = _oracle_blocks(port, sb, r, Hq, Hkv, cfg)
        _assert_blocks_close(bs[cub[r]:cub[r + 1]], want)


_PACK_CHILD = r'''
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import oracle, paper_2605_06221_b200 as up
from paper_2605_06221_b200.synthetic import make_batch
port = oracle.port()
bad = []
for Hq, Hkv, D, lengths, n, G in [(8, 2, 128, [1000, 2000, 40], 32, 64),    # GQA 4: 2 heads per tile
                                  (8, 2, 128, [1500, 63], 64, 32),          # n = 64
                                  (16, 2, 256, [3000, 700], 32, 64),        # Qwen3-Next heads: 4 per tile
                                  (8, 2, 128, [900, 5], 20, 64),            # npad 32, short requests
                                  (8, 2, 128, [777], 1, 64)]:               # n = 1
    cfg = dict(query_window_n=n, block_size_g=G, sink_count_a=128, top_p=0.99)
    sb = make_batch(lengths, Hq, Hkv, D, 64, regime="planted", block_size_g=G, seed=sum(lengths) + 3 * n)
    res = up.score_blocks_varlen(sb.q, sb.k, sb.cu_seqlens, up.ScoreConfig(**cfg), up.HeadLayout(Hq, Hkv, D), check=True)
    cu, cub, bs = sb.cu_seqlens.cpu().numpy(), res.cu_blocks.cpu().numpy(), res.block_scores.cpu().numpy().astype(np.float64)
    for r in range(len(lengths)):
        s, e = int(cu[r]), int(cu[r + 1])
        _, want, _ = port.score_tokens(sb.q[s:e].float().reshape(e - s, -1).cpu().numpy(),
                                       sb.k[s:e].float().reshape(e - s, -1).cpu().numpy(), Hq, Hkv, **cfg)
        got = bs[cub[r]:cub[r + 1]]
        atol = 1e-6 * max(want.sum(), 1e-30) / len(want)
        if len(got) != len(want) or (np.abs(got - want) > 1e-3 * np.abs(want) + atol).any():
            bad.append((Hq, Hkv, D, lengths, n, G, r))
print("PACK_BAD", bad)
'''


def test_short_query_window_packs_heads_into_one_tile(up):
    """n <= 64 (the paper's n = 32 ablation): P q-heads of a kv-group share one 128-row S
    tile (score_tcw's TS variant loads each row's Q from its own head), so a 32-row window
    does not pay for 128 rows.  Block scores vs the oracle within rtol 1e-3; the child
    process asserts packing served every call."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", _PACK_CHILD, root], capture_output=True, text=True, timeout=900,
                         env=dict(os.environ, UP_SCORE_VERBOSE="1"))
    assert out.returncode == 0, out.stderr[-2000:]
    assert "pack=1" not in out.stderr and "pack=" in out.stderr
    assert "PACK_BAD []" in out.stdout, out.stdout[-2000:]


_PW_CHILD = r'''
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_2605_06221_b200 as up
from paper_2605_06221_b200.synthetic import make_batch
out = []
for Hq, Hkv, D, lengths in [(32, 8, 128, [100] * 300 + [9000]),     # HPC 4: one-item pairs + a spread pair
                            (8, 8, 128, [90] * 200 + [130, 5000]),  # HPC 1, four parity rows
                            (16, 2, 256, [200] * 50 + [3000])]:     # HPC 2 TS
    sb = make_batch(lengths, Hq, Hkv, D, 64, regime="planted", seed=len(lengths) + D)
    res = up.score_blocks_varlen(sb.q, sb.k, sb.cu_seqlens, up.ScoreConfig(), up.HeadLayout(Hq, Hkv, D), check=True)
    torch.cuda.synchronize()
    out.append(res.block_scores[:int(res.cu_blocks[-1])].cpu().numpy().view(np.uint32))
np.save(sys.argv[2], np.concatenate(out))
'''


def test_pair_weights_warp_path_is_bitwise_the_cta_path(up, tmp_path):
    """pair_weights does pairs held by <= 2 scorer CTAs one warp each and wider pairs one
    CTA each, with the same arithmetic (each item's parity rows folded from (-inf, 0), the
    items merged in order): block scores are bitwise identical when every pair is forced
    down the CTA path (UP_PW_WARP_ITEMS=0, child processes: read once per process)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    got = {}
    for wi in ("2", "0"):
        f = str(tmp_path / f"pw_{wi}.npy")
        r = subprocess.run([sys.executable, "-c", _PW_CHILD, root, f], capture_output=True, text=True, timeout=600,
                           env=dict(os.environ, UP_PW_WARP_ITEMS=wi))
        assert r.returncode == 0, r.stderr[-2000:]
        got[wi] = np.load(f)
    assert got["2"].size > 0 and np.array_equal(got["2"], got["0"])
