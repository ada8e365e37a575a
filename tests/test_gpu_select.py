"""GPU parity: top-p keep mask vs the reference (selection.cpp:14-122), bit-exact.

Cases restate /root/reference/proj/tests/test_selection.cpp and acceptance criterion 3
(acceptance_main.cpp:175-217); every random vector is also checked against the C oracle.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def plain(up, p, g=1, a=0, n=1):
    return up.ScoreConfig(query_window_n=n, block_size_g=g, sink_count_a=a, top_p=p)


def _cfgd(c):
    return dict(query_window_n=c.query_window_n, block_size_g=c.block_size_g,
                sink_count_a=c.sink_count_a, top_p=c.top_p)


def _same(up, port, scores, cfg, N, veto=None):
    scores = np.asarray(scores, np.float32)
    sel = up.top_p_select(torch.from_numpy(scores).cuda(), cfg, N,
                          veto=None if veto is None else torch.from_numpy(veto).cuda())
    want = port.top_p_select(scores, N, **_cfgd(cfg))
    if veto is not None:
        want = port.restrict_selection(want, veto, scores, cfg.block_size_g)
    got = sel.keep_mask.cpu().numpy()
    assert np.array_equal(got, want.keep_mask), (np.flatnonzero(got != want.keep_mask)[:10])
    assert sel.cutoff_rank == want.cutoff_rank
    assert sel.retained_count() == want.retained_count
    assert np.array_equal(sel.retained_indices.cpu().numpy(), want.retained_indices)
    assert sel.degenerate_keep_all == want.degenerate_keep_all
    assert abs(sel.covered_mass - want.covered_mass) <= 1e-12 * max(1.0, abs(want.covered_mass))
    return sel


def test_worked_example(up, port):
    sel = _same(up, port, [0.5, 0.3, 0.15, 0.05], plain(up, 0.9), 4)
    assert sel.cutoff_rank == 3
    assert sel.keep_mask.cpu().tolist() == [1, 1, 1, 1]


def test_top_p_one_keeps_everything(up, port):
    sel = _same(up, port, [0.9, 0.05, 0.04, 0.01], plain(up, 1.0), 4)
    assert sel.cutoff_rank == 4 and sel.retention_ratio == 1.0


def test_uniform_keeps_all_ten(up, port):
    sel = _same(up, port, [0.1] * 10, plain(up, 0.99), 10)
    assert sel.cutoff_rank == 10 and sel.retained_count() == 10


def test_zero_mass_degenerates(up, port):
    sel = _same(up, port, [0.0] * 5, plain(up, 0.5), 5)
    assert sel.degenerate_keep_all and sel.retained_count() == 5 and sel.covered_mass == 1.0


def test_negative_or_nan_rejected(up):
    with pytest.raises(up.ContractViolation):
        up.top_p_select(torch.tensor([0.5, -0.1]).cuda(), plain(up, 0.9), 2)
    with pytest.raises(up.ContractViolation):
        up.top_p_select(torch.tensor([0.5, float("nan")]).cuda(), plain(up, 0.9), 2)
    with pytest.raises(up.ContractViolation):
        up.top_p_select(torch.tensor([0.5, float("inf")]).cuda(), plain(up, 0.9), 2)


def test_config_errors(up):
    for bad in (plain(up, 0.0), plain(up, 1.5), up.ScoreConfig(0, 64, 1, 0.9),
                up.ScoreConfig(8, 0, 1, 0.9), up.ScoreConfig(8, 8, -1, 0.9)):
        with pytest.raises(up.ConfigError):
            up.top_p_select(torch.tensor([1.0]).cuda(), bad, 1)


def test_concentrated_and_uniform_adaptivity(up, port):
    conc = [0.0001] * 20
    conc[7] = 1.0
    sel = _same(up, port, conc, plain(up, 0.9), 20)
    assert sel.cutoff_rank == 1 and bool(sel.keep_mask[7].item())
    sel = _same(up, port, [1.0] * 50, plain(up, 0.99), 50)
    assert sel.cutoff_rank == 50


def test_ties_prefer_lower_index(up, port):
    scores = np.array([0.25, 0.5, 0.25, 0.25, 0.5, 0.0, 0.25], np.float32)
    for p in (0.3, 0.5, 0.6, 0.75, 0.8, 0.95):
        _same(up, port, scores, plain(up, p), len(scores))


def test_random_vectors_match_oracle(up, port):
    """test_selection.cpp:201-231 style: zeros, quantised ties, denormals, uniforms."""
    rng = np.random.default_rng(21)
    for trial in range(300):
        nb = int(rng.integers(1, 81))
        kind = rng.integers(0, 4, nb)
        s = rng.random(nb).astype(np.float32)
        s[kind == 0] = 0.0
        s[kind == 1] = (np.floor(rng.random((kind == 1).sum()) * 4) * 0.25).astype(np.float32)
        s[kind == 2] = np.float32(1.4e-45) * rng.integers(1, 6, (kind == 2).sum()).astype(np.float32)
        p = 1.0 if trial % 3 == 0 else float(np.float32(0.5 + 0.49 * rng.random()))
        _same(up, port, s, plain(up, p), nb)


def test_acceptance_c3_sample(up, port):
    """Acceptance criterion 3 (acceptance_main.cpp:175-217): log-uniform lengths to 4096."""
    rng = np.random.default_rng(31)
    for trial in range(400):
        n = max(1, int(2.0 ** (rng.random() * 12.0)))
        kind = rng.integers(0, 5, n)
        s = rng.random(n).astype(np.float32)
        s[kind == 0] = 0.0
        m = kind == 1
        s[m] = (np.floor(rng.random(m.sum()) * 8) * 0.125).astype(np.float32)
        m = kind == 2
        s[m] = np.float32(1.4e-45) * rng.integers(1, 8, m.sum()).astype(np.float32)
        p = 1.0 if trial % 7 == 0 else float(np.float32(0.3 + 0.7 * rng.random()))
        _same(up, port, s, plain(up, p), n)


def test_blocks_sinks_window_and_veto(up, port):
    """covered_mass >= p with forced sinks/window (test_selection.cpp:290-317) + veto."""
    rng = np.random.default_rng(24)
    for trial in range(50):
        N = 40 + int(rng.integers(0, 200))
        cfg = up.ScoreConfig(query_window_n=8, block_size_g=8, sink_count_a=8, top_p=0.8)
        nb = (N + 7) // 8
        s = (rng.random(nb) * rng.random(nb)).astype(np.float32)
        sel = _same(up, port, s, cfg, N)
        assert sel.covered_mass >= 0.8 - 1e-12
        veto = (rng.random(N) < 0.2).astype(np.uint8)
        _same(up, port, s, cfg, N, veto=veto)


def test_scale_invariance(up, port):
    rng = np.random.default_rng(23)
    s = rng.random(33).astype(np.float32)
    cfg = plain(up, 0.85, 1, 2, 3)
    base = _same(up, port, s, cfg, 33)
    for c in (0.25, 0.5, 2.0, 1024.0, 2.0 ** -20):
        moved = _same(up, port, (s * np.float32(c)).astype(np.float32), cfg, 33)
        assert torch.equal(moved.keep_mask, base.keep_mask)
        assert moved.cutoff_rank == base.cutoff_rank


def test_varlen_select_matches_per_request(up, port):
    rng = np.random.default_rng(5)
    lengths = [4096, 1, 130, 64, 2000, 65]
    G = 64
    cfg = up.ScoreConfig()
    nbs = [(n + G - 1) // G for n in lengths]
    scores = [rng.random(nb).astype(np.float32) ** 8 for nb in nbs]
    cu = np.concatenate([[0], np.cumsum(lengths)]).astype(np.int32)
    cub = np.concatenate([[0], np.cumsum(nbs)]).astype(np.int32)
    en = np.array([1, 1, 1, 0, 1, 1], np.uint8)
    sel = up.select_varlen(torch.from_numpy(np.concatenate(scores)).cuda(), torch.from_numpy(cub).cuda(),
                           torch.from_numpy(cu).cuda(), cfg, drop_enabled=torch.from_numpy(en).cuda(),
                           check=True)
    keep = sel.keep.cpu().numpy()
    for r, n in enumerate(lengths):
        got = keep[cu[r]:cu[r + 1]]
        if not en[r]:
            assert got.all() and int(sel.cutoff_rank[r]) == -1
            continue
        want = port.top_p_select(scores[r], n, **_cfgd(cfg))
        assert np.array_equal(got, want.keep_mask)
        assert int(sel.cutoff_rank[r]) == want.cutoff_rank


def test_request_beyond_2048_blocks_uses_bitonic_kernel(up, port):
    """A 200K-token request (3125 blocks) goes to the large-request select kernel; the keep
    mask and k* stay bit-exact with the reference; a small request in the same batch is
    served by the small size class."""
    rng = np.random.default_rng(21)
    lengths = [200000, 3000]
    G = 64
    nbs = [(n + G - 1) // G for n in lengths]
    scores = (rng.random(sum(nbs)) ** 6).astype(np.float32)
    cu = torch.tensor(np.concatenate([[0], np.cumsum(lengths)]), dtype=torch.int32, device="cuda")
    cub = torch.tensor(np.concatenate([[0], np.cumsum(nbs)]), dtype=torch.int32, device="cuda")
    cfg = dict(query_window_n=128, block_size_g=G, sink_count_a=128, top_p=0.99)
    sel = up.select_varlen(torch.from_numpy(scores).cuda(), cub, cu, up.ScoreConfig(**cfg), check=True)
    keep = sel.keep.cpu().numpy()
    kst = sel.cutoff_rank.cpu().numpy()
    off = 0
    for r, n in enumerate(lengths):
        want = port.top_p_select(scores[sum(nbs[:r]):sum(nbs[:r + 1])], n, **cfg)
        assert np.array_equal(keep[off:off + n], want.keep_mask)
        assert int(kst[r]) == want.cutoff_rank
        off += n


def test_every_size_class_in_one_batch_eager_and_graph(up, port):
    """One batch holding every select path: direct ranks (<= 128 blocks), radix select
    (<= 512), the 512-thread sort (<= 2048, side stream) and the bitonic kernel (> 2048,
    side stream), plus a single-token request -- bit-exact with the reference eagerly and
    replayed from a CUDA graph (the side stream's fork / join captured as graph edges)."""
    rng = np.random.default_rng(33)
    lengths = [150000, 60000, 20000, 3000, 100, 1]
    G = 64
    nbs = [(n + G - 1) // G for n in lengths]
    scores = (rng.random(sum(nbs)) ** 7).astype(np.float32)
    cu = torch.tensor(np.concatenate([[0], np.cumsum(lengths)]), dtype=torch.int32, device="cuda")
    cub = torch.tensor(np.concatenate([[0], np.cumsum(nbs)]), dtype=torch.int32, device="cuda")
    cfgd = dict(query_window_n=128, block_size_g=G, sink_count_a=128, top_p=0.99)
    cfg = up.ScoreConfig(**cfgd)
    d_scores = torch.from_numpy(scores).cuda()
    sel = up.select_varlen(d_scores, cub, cu, cfg, check=True)
    want_keep = []
    for r, n in enumerate(lengths):
        w = port.top_p_select(scores[sum(nbs[:r]):sum(nbs[:r + 1])], n, **cfgd)
        want_keep.append(w.keep_mask)
        assert int(sel.cutoff_rank[r]) == w.cutoff_rank
    want_keep = np.concatenate(want_keep)
    T = sum(lengths)
    assert np.array_equal(sel.keep[:T].cpu().numpy(), want_keep)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        up.select_varlen(d_scores, cub, cu, cfg, out=sel, max_tokens=T)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            with pytest.raises(up.ContractViolation):  # the capacity must come from the caller
                up.select_varlen(d_scores, cub, cu, cfg, out=sel)
            up.select_varlen(d_scores, cub, cu, cfg, out=sel, max_tokens=T)
        sel.keep.zero_()
        g.replay()
    torch.cuda.synchronize()
    assert np.array_equal(sel.keep[:T].cpu().numpy(), want_keep)


def test_maximum_request_size(up, port):
    """The largest request the on-chip sort holds: 2^20 tokens = 16384 blocks of 64 (a 1M
    context), bit-exact with the reference; one block more raises the sticky
    UnsupportedError (and keeps the request whole rather than dropping anything)."""
    rng = np.random.default_rng(5)
    G = 64
    cfg = dict(query_window_n=128, block_size_g=G, sink_count_a=128, top_p=0.99)
    n = 1 << 20
    nb = n // G
    scores = (rng.random(nb) ** 8).astype(np.float32)
    cu = torch.tensor([0, n], dtype=torch.int32, device="cuda")
    cub = torch.tensor([0, nb], dtype=torch.int32, device="cuda")
    sel = up.select_varlen(torch.from_numpy(scores).cuda(), cub, cu, up.ScoreConfig(**cfg), check=True)
    want = port.top_p_select(scores, n, **cfg)
    assert np.array_equal(sel.keep.cpu().numpy(), want.keep_mask)
    assert int(sel.cutoff_rank[0]) == want.cutoff_rank

    n2 = n + 1
    scores2 = np.concatenate([scores, scores[:1]])
    cu2 = torch.tensor([0, n2], dtype=torch.int32, device="cuda")
    cub2 = torch.tensor([0, nb + 1], dtype=torch.int32, device="cuda")
    ws = up.Workspace("cuda")
    sel2 = up.select_varlen(torch.from_numpy(scores2).cuda(), cub2, cu2, up.ScoreConfig(**cfg), workspace=ws)
    with pytest.raises(up.UnsupportedError):
        ws.device_status()
    assert bool(sel2.keep.bool().all())
