"""GPU parity: segmented prefix sum + gather compaction (propagation.cpp:47-77,
scheduler.cpp:50-90), byte-exact against the oracle and the reference's own KATs."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _sel(up, keep):
    keep = torch.tensor(keep, dtype=torch.uint8, device="cuda")
    idx = torch.nonzero(keep).flatten()
    return up.Selection(keep, idx, idx.numel() / keep.numel(), 1.0, idx.numel(), False)


def test_apply_drop_keep_all_identity(up):
    prompt = torch.randn(6, 32, device="cuda")
    stream = up.TokenStream.from_prompt(prompt)
    hist = up.DropHistory(original_length=6)
    up.apply_drop(stream, _sel(up, [1] * 6), 0, hist)
    assert stream.active_count() == 6
    assert torch.equal(stream.active_states, prompt)
    assert not stream.parked_states
    assert hist.events[0].retained_length == 6


def test_apply_drop_compaction_order(up):
    prompt = torch.randn(8, 32, device="cuda")
    stream = up.TokenStream.from_prompt(prompt)
    hist = up.DropHistory(original_length=8)
    up.apply_drop(stream, _sel(up, [1, 1, 0, 0, 0, 0, 1, 1]), 0, hist)
    assert stream.logical_positions.tolist() == [0, 1, 6, 7]
    assert torch.equal(stream.active_states[2], prompt[6])
    assert stream.parked_positions[0].tolist() == [2, 3, 4, 5]
    assert torch.equal(stream.parked_states[0][1], prompt[3])


def test_stacked_drops_compose(up):
    prompt = torch.randn(8, 32, device="cuda")
    stream = up.TokenStream.from_prompt(prompt)
    hist = up.DropHistory(original_length=8)
    m1 = [1, 1, 0, 1, 1, 0, 1, 1]
    up.apply_drop(stream, _sel(up, m1), 0, hist)
    m2 = [1, 0, 1, 0, 1, 1]
    up.apply_drop(stream, _sel(up, m2), 4, hist)
    first = [i for i in range(8) if m1[i]]
    survivors = [first[i] for i in range(len(first)) if m2[i]]
    assert stream.logical_positions.tolist() == survivors
    parked = sorted(int(x) for p in stream.parked_positions for x in p.tolist())
    assert parked == sorted(set(range(8)) - set(survivors))
    assert hist.events[1].retained_length == len(survivors)


def test_patch_metadata_kats(up):
    """test_scheduler.cpp:154-203."""
    toks = torch.randn(16, 8, device="cuda")
    b = up.PackedBatch(toks.clone(), torch.tensor([0, 8, 16]), ["prefill", "prefill"])
    up.patch_metadata(b, [None, None], 0)
    assert b.cu_seqlens.tolist() == [0, 8, 16] and torch.equal(b.tokens, toks)

    b = up.PackedBatch(toks.clone(), torch.tensor([0, 8, 16]), ["prefill", "prefill"])
    up.patch_metadata(b, [_sel(up, [1, 0, 1, 0, 1, 0, 1, 0]), None], 0)
    assert b.cu_seqlens.tolist() == [0, 4, 12]
    assert torch.equal(b.tokens[1], toks[2]) and torch.equal(b.tokens[4], toks[8])

    t9 = torch.randn(9, 8, device="cuda")
    b = up.PackedBatch(t9, torch.tensor([0, 8, 9]), ["prefill", "decode"])
    up.patch_metadata(b, [_sel(up, [1, 1, 1, 1, 0, 0, 0, 0]), None], 0)
    assert b.cu_seqlens.tolist() == [0, 4, 5]
    with pytest.raises(up.ContractViolation):
        up.patch_metadata(b, [None, _sel(up, [0])], 1)


@pytest.mark.parametrize("lengths,row_bytes", [
    ([1000, 1, 77, 4096, 3], (8192, 2048, 2048, 8)),
    ([300], (4096, 512, 4)),
    ([5, 2049, 513], (16, 24, 6)),   # odd row sizes exercise the narrow copy paths
])
def test_compact_matches_oracle(up, port, lengths, row_bytes):
    rng = np.random.default_rng(len(lengths))
    T = sum(lengths)
    cu = np.concatenate([[0], np.cumsum(lengths)]).astype(np.int64)
    keep = (rng.random(T) < 0.3).astype(np.uint8)
    en = (rng.random(len(lengths)) < 0.8).astype(np.uint8)
    planes = [rng.integers(0, 255, (T, rb), dtype=np.uint8) for rb in row_bytes]
    want, cu_want, idx_want = port.compact(keep, cu, planes, selected=en)
    res = up.compact_varlen(torch.from_numpy(keep).cuda(), torch.from_numpy(cu).cuda(),
                            [torch.from_numpy(p).cuda() for p in planes],
                            drop_enabled=torch.from_numpy(en).cuda(), check=True).trimmed()
    assert res.cu_seqlens.cpu().tolist() == cu_want.tolist()
    assert np.array_equal(res.retained_index.cpu().numpy(), idx_want)
    for g, w in zip(res.planes, want):
        assert np.array_equal(g.cpu().numpy(), w)


def test_compact_capacity_larger_than_batch(up, port):
    """max_tokens capacity > cu[R]: rows past the batch are ignored."""
    lengths = [500, 700]
    T = 1200
    cap = 4000
    rng = np.random.default_rng(9)
    keep = np.zeros(cap, np.uint8)
    keep[:T] = (rng.random(T) < 0.5)
    hid = torch.randn(cap, 64, device="cuda").to(torch.bfloat16)
    cu = torch.tensor([0, 500, 1200], dtype=torch.int32, device="cuda")
    res = up.compact_varlen(torch.from_numpy(keep).cuda(), cu, [hid], max_tokens=cap, check=True)
    n = int(res.num_out.item())
    assert n == int(keep[:T].sum())
    idx = np.flatnonzero(keep[:T])
    assert torch.equal(res.planes[0][:n], hid[torch.from_numpy(idx).cuda()])
    assert res.cu_seqlens.cpu().tolist() == [0, int(keep[:500].sum()), n]


def test_compact_reads_pinned_host_planes_in_place(up):
    """Source planes in pinned host memory are gathered in place (zero-copy over PCIe):
    byte-identical to compacting the same planes from device memory."""
    g = torch.Generator().manual_seed(9)
    lengths = [3000, 1, 1700]
    T = sum(lengths)
    cu = torch.tensor(np.concatenate([[0], np.cumsum(lengths)]), dtype=torch.int32, device="cuda")
    keep = (torch.rand(T, generator=g) < 0.3).to(torch.uint8).cuda()
    hid_h = torch.randn(T, 4096, generator=g).to(torch.bfloat16).pin_memory()
    v_h = torch.randn(T, 2, 128, generator=g).to(torch.bfloat16).pin_memory()
    pos_h = torch.arange(T, dtype=torch.int64).pin_memory()
    k_d = torch.randn(T, 2, 128, generator=g).to(torch.bfloat16).cuda()
    outs = [torch.empty(T, 4096, dtype=torch.bfloat16, device="cuda"), torch.empty_like(k_d),
            torch.empty(T, 2, 128, dtype=torch.bfloat16, device="cuda"),
            torch.empty(T, dtype=torch.int64, device="cuda")]
    res = up.compact_varlen(keep, cu, [hid_h, k_d, v_h, pos_h], outs=outs, check=True)
    want = up.compact_varlen(keep, cu, [hid_h.cuda(), k_d, v_h.cuda(), pos_h.cuda()], check=True)
    n = int(res.num_out.item())
    assert n == int(want.num_out.item()) == int(keep.sum().item())
    assert torch.equal(res.cu_seqlens, want.cu_seqlens)
    for a, b in zip(res.planes, want.planes):
        assert torch.equal(a[:n], b[:n])
    with pytest.raises(up.ContractViolation):  # pageable host memory is rejected
        up.compact_varlen(keep, cu, [torch.zeros(T, 8)], outs=[torch.empty(T, 8, device="cuda")])


def _ref_reconstitute(ref, prompt, keeps, afters):
    return ref.reconstitute_sequence(prompt, keeps, afters)


@pytest.mark.parametrize("rows,drops", [(1, 1), (8, 2), (300, 3), (2049, 2)])
def test_reconstitute_matches_reference(up, ref, rows, drops):
    """TokenStream: apply_drop x k (states transformed in between) then reconstitute ==
    the reference's reconstitute (propagation.cpp:79-100), bit for bit."""
    rng = np.random.default_rng(rows * 10 + drops)
    cols = 24
    prompt = rng.standard_normal((rows, cols)).astype(np.float32)
    stream = up.TokenStream.from_prompt(torch.from_numpy(prompt).cuda())
    hist = up.DropHistory(original_length=rows)
    keeps, afters = [], []
    for d in range(drops):
        n = stream.active_count()
        keep = (rng.random(n) < 0.6).astype(np.uint8)
        keep[0] = 1  # keep the stream non-empty
        up.apply_drop(stream, _sel(up, keep.tolist()), d, hist)
        after = rng.standard_normal((int(keep.sum()), cols)).astype(np.float32)
        stream.active_states = torch.from_numpy(after).cuda()
        keeps.append(keep)
        afters.append(after)
    up.reconstitute(stream)
    want_states, want_pos = _ref_reconstitute(ref, prompt, keeps, afters)
    assert stream.logical_positions.cpu().tolist() == want_pos.tolist()
    assert np.array_equal(stream.active_states.cpu().numpy().view(np.uint32), want_states.view(np.uint32))
    assert not stream.parked_states
    up.reconstitute(stream)  # idempotent without parked rows
    assert np.array_equal(stream.active_states.cpu().numpy(), want_states)


def test_reconstitute_varlen_unwinds_drops_in_reverse(up, ref):
    """Varlen batch: two out-of-place drops (compact_varlen), states transformed after each,
    then the block boundary unwinds them with reconstitute_varlen (scatter of the compacted
    rows over the pre-drop buffers) -> every request equals the reference reconstitute."""
    rng = np.random.default_rng(4)
    lengths = [700, 1, 1300, 64]
    R, T, cols = len(lengths), sum(lengths), 32
    cu0 = torch.tensor(np.concatenate([[0], np.cumsum(lengths)]), dtype=torch.int32, device="cuda")
    prompt = rng.standard_normal((T, cols)).astype(np.float32)
    buf0 = torch.from_numpy(prompt).cuda()               # pre-drop buffer of drop 0
    keep0 = (rng.random(T) < 0.5).astype(np.uint8)
    c0 = up.compact_varlen(torch.from_numpy(keep0).cuda(), cu0, [buf0], check=True)
    n0 = int(c0.num_out.item())
    after0 = rng.standard_normal((n0, cols)).astype(np.float32)
    buf1 = torch.from_numpy(after0).cuda()               # states entering drop 1 (= pre-drop buffer 1)
    keep1 = (rng.random(n0) < 0.5).astype(np.uint8)
    c1 = up.compact_varlen(torch.from_numpy(keep1).cuda(), c0.cu_seqlens, [buf1], max_tokens=n0, check=True)
    n1 = int(c1.num_out.item())
    after1 = rng.standard_normal((n1, cols)).astype(np.float32)
    cur = torch.from_numpy(after1).cuda()              # the layers after drop 1 transform the stream
    up.reconstitute_varlen([cur], c1, [buf1])           # unwind drop 1: buf1 = stream in drop-0 row space
    up.reconstitute_varlen([buf1], c0, [buf0])          # then drop 0: buf0 is the full stream
    got = buf0.cpu().numpy()
    cu0h, cu1h, cu2h = cu0.cpu().numpy(), c0.cu_seqlens.cpu().numpy(), c1.cu_seqlens.cpu().numpy()
    for r in range(R):
        s, e = cu0h[r], cu0h[r + 1]
        k0 = keep0[s:e]
        k1 = keep1[cu1h[r]:cu1h[r + 1]]
        a0 = after0[cu1h[r]:cu1h[r + 1]]
        a1 = after1[cu2h[r]:cu2h[r + 1]]
        want, pos = _ref_reconstitute(ref, prompt[s:e], [k0, k1], [a0, a1]) if k0.any() and k1.any() else (None, None)
        if want is None:
            continue
        assert np.array_equal(got[s:e].view(np.uint32), want.view(np.uint32)), f"request {r}"


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_compact_after_select_matches_full_scan(up, seed):
    """up_compact_selected (the tile counts come from up_select's expansion) equals up_compact
    on the same keep mask: drop-disabled segments, a veto, lengths across tile boundaries."""
    rng = np.random.default_rng(seed)
    lengths = [int(x) for x in rng.choice([1, 63, 1023, 1024, 1025, 3000, 5000], size=5)]
    T, R = sum(lengths), len(lengths)
    G = 64
    nbs = [(n + G - 1) // G for n in lengths]
    scores = torch.from_numpy((rng.random(sum(nbs)) ** 8).astype(np.float32)).cuda()
    cu = torch.tensor(np.concatenate([[0], np.cumsum(lengths)]), dtype=torch.int32, device="cuda")
    cub = torch.tensor(np.concatenate([[0], np.cumsum(nbs)]), dtype=torch.int32, device="cuda")
    en = torch.from_numpy((rng.random(R) < 0.7).astype(np.uint8)).cuda()
    veto = torch.from_numpy((rng.random(T) < 0.05).astype(np.uint8)).cuda()
    ws = up.Workspace("cuda")
    cfg = up.ScoreConfig(top_p=0.9)
    sel = up.select_varlen(scores, cub, cu, cfg, veto=veto, drop_enabled=en, workspace=ws, check=True)
    hid = torch.randn(T, 48, device="cuda").to(torch.bfloat16)
    pos = torch.arange(T, dtype=torch.int64, device="cuda")
    a = up.compact_varlen(sel.keep, cu, [hid, pos], drop_enabled=en, workspace=ws, after_select=True, check=True)
    b = up.compact_varlen(sel.keep, cu, [hid, pos], drop_enabled=en, check=True)
    n = int(b.num_out.item())
    assert int(a.num_out.item()) == n
    assert torch.equal(a.cu_seqlens, b.cu_seqlens)
    assert torch.equal(a.retained_index[:n], b.retained_index[:n])
    for x, y in zip(a.planes, b.planes):
        assert torch.equal(x[:n], y[:n])


@pytest.mark.parametrize("seed", [3, 4])
def test_small_capacity_paths_match_large(up, seed):
    """At capacities <= 8192 rows the select CTAs expand their own token masks (no
    expand_kernel launch) and compaction is one launch (compact_small_kernel); the same
    batch under a larger capacity takes the grid-wide expand + count/index/copy kernels.
    Both must give identical keep masks, selections and compacted outputs (drop-disabled
    segments, a veto, lengths across the 1024-row tiles)."""
    rng = np.random.default_rng(seed)
    lengths = [int(x) for x in rng.choice([1, 63, 700, 1024, 1025, 2000], size=4)]
    T, R = sum(lengths), len(lengths)
    assert T <= 8192
    G = 64
    nbs = [(n + G - 1) // G for n in lengths]
    scores = torch.from_numpy((rng.random(sum(nbs)) ** 8).astype(np.float32)).cuda()
    cu = torch.tensor(np.concatenate([[0], np.cumsum(lengths)]), dtype=torch.int32, device="cuda")
    cub = torch.tensor(np.concatenate([[0], np.cumsum(nbs)]), dtype=torch.int32, device="cuda")
    en = torch.from_numpy((rng.random(R) < 0.75).astype(np.uint8)).cuda()
    veto = torch.from_numpy((rng.random(T) < 0.05).astype(np.uint8)).cuda()
    cfg = up.ScoreConfig(top_p=0.9)
    hid = torch.randn(T, 40, device="cuda").to(torch.bfloat16)
    pos = torch.arange(T, dtype=torch.int64, device="cuda")
    outs = []
    for cap in (T, T + 9000):
        ws = up.Workspace("cuda")
        sc = torch.zeros(cap // G + R + 1, dtype=torch.float32, device="cuda")
        sc[:scores.numel()] = scores
        sel = up.select_varlen(sc, cub, cu, cfg, veto=veto, drop_enabled=en, max_tokens=cap, workspace=ws,
                               check=True)
        n_sel = up.lib.up_last_launch_count()
        planes = [torch.cat([hid, torch.zeros(cap - T, 40, dtype=hid.dtype, device="cuda")]),
                  torch.cat([pos, torch.zeros(cap - T, dtype=pos.dtype, device="cuda")])]
        c = up.compact_varlen(sel.keep, cu, planes, drop_enabled=en, max_tokens=cap, workspace=ws,
                              after_select=True, check=True)
        n_cmp = up.lib.up_last_launch_count()
        outs.append((sel, c, n_sel, n_cmp))
    (s0, c0, ns0, nc0), (s1, c1, ns1, nc1) = outs
    assert (ns0, nc0) == (1, 1) and ns1 >= 2 and nc1 >= 2  # the small paths actually ran
    assert torch.equal(s0.keep[:T], s1.keep[:T])
    assert torch.equal(s0.cutoff_rank, s1.cutoff_rank)
    n = int(c1.num_out.item())
    assert int(c0.num_out.item()) == n
    assert torch.equal(c0.cu_seqlens, c1.cu_seqlens)
    assert torch.equal(c0.retained_index[:n], c1.retained_index[:n])
    for x, y in zip(c0.planes, c1.planes):
        assert torch.equal(x[:n], y[:n])
