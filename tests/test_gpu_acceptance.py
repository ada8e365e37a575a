"""GPU: the reference's own acceptance gates for the hot path, at their full size.

* c3 (acceptance_main.cpp:175-217): all 100,000 random score vectors of the criterion's
  CounterRng(31, 0x6333) stream (lengths 1-4096 log-uniform, zeros, quantised ties,
  subnormals; p = 1 every 7th trial) through up_select, one R = 1 launch each (top_p differs
  per vector), keep masks and k* bit-exact against the reference's top_p_select -- which
  tests/test_oracle.py pins against the criterion's sort-and-cumsum oracle.
* c8 (acceptance_main.cpp:445-478): its 100 q/k inputs (H = 8, D = 8, n = G = A = 8,
  p = 0.9) rounded to bf16, scored head-sharded through up_score_blocks_tp for
  T in {1, 2, 4, 8} and selected: identical selections for every T, and against the
  reference (same bf16-exact inputs) block scores within rtol 1e-3 and keep masks equal
  outside the tie band.
"""
import ctypes

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

RTOL = 1e-3


@pytest.fixture(scope="module")
def checker(port):
    import oracle
    return oracle.ref() if oracle.ref_available() else None


@pytest.mark.timeout(900)
def test_acceptance_c3_all_100k_vectors(up, port, checker):
    from paper_2605_06221_b200 import _capi
    from paper_2605_06221_b200.api import _stream_ptr
    s, off, ps = port.c3_vectors(100000)
    T = len(ps)
    if checker is not None:
        want, want_cut = checker.top_p_select_batch(s, off, ps, query_window_n=1, block_size_g=1, sink_count_a=0)
    else:  # the port, pinned to the reference by tests/test_oracle.py
        sels = [port.top_p_select(s[off[t]:off[t + 1]], int(off[t + 1] - off[t]), query_window_n=1,
                                  block_size_g=1, sink_count_a=0, top_p=float(ps[t])) for t in range(T)]
        want = np.concatenate([x.keep_mask for x in sels])
        want_cut = np.array([x.cutoff_rank for x in sels], np.int64)
    lens = (off[1:] - off[:-1]).astype(np.int32)
    cu = torch.zeros((T, 2), dtype=torch.int32)
    cu[:, 1] = torch.from_numpy(lens)
    cu = cu.cuda()
    scores = torch.from_numpy(s).cuda()
    keep = torch.full((len(s),), 7, dtype=torch.uint8, device="cuda")
    cut = torch.empty(T, dtype=torch.int64, device="cuda")
    ret = torch.empty(T, dtype=torch.int64, device="cuda")
    cov = torch.empty(T, dtype=torch.float64, device="cuda")
    deg = torch.empty(T, dtype=torch.uint8, device="cuda")
    lib = up.lib
    big = _capi.BatchC(1, 4096, ctypes.c_void_p(cu.data_ptr()), None)
    ws = torch.zeros(int(lib.up_workspace_bytes(ctypes.byref(big), None,
                                                ctypes.byref(_capi.ScoreConfigC(1, 1, 0, 0.9)))),
                     dtype=torch.uint8, device="cuda")
    stream = _stream_ptr("cuda")
    sp, kp, cp = scores.data_ptr(), keep.data_ptr(), cu.data_ptr()
    for t in range(T):
        b = _capi.BatchC(1, int(lens[t]), ctypes.c_void_p(cp + 8 * t), None)
        c = _capi.ScoreConfigC(1, 1, 0, float(ps[t]))
        so = _capi.SelectionOutC(cut.data_ptr() + 8 * t, ret.data_ptr() + 8 * t, cov.data_ptr() + 8 * t,
                                 deg.data_ptr() + t)
        # G = 1: cu_blocks == cu_seqlens
        st = lib.up_select(stream, ctypes.byref(b), ctypes.byref(c), ctypes.c_void_p(sp + 4 * int(off[t])),
                           ctypes.c_void_p(cp + 8 * t), None, ctypes.c_void_p(kp + int(off[t])), ctypes.byref(so),
                           ctypes.c_void_p(ws.data_ptr()), ws.numel())
        assert st == 0, (t, st)
    torch.cuda.synchronize()
    assert lib.up_device_status(stream, ctypes.c_void_p(ws.data_ptr())) == 0
    got = keep.cpu().numpy()
    bad = np.flatnonzero(got != want)
    assert bad.size == 0, f"{bad.size} keep bytes differ; first trials " \
        f"{sorted(set(np.searchsorted(off, bad[:20], side='right') - 1))}"
    assert np.array_equal(cut.cpu().numpy(), want_cut)
    assert np.array_equal(ret.cpu().numpy(), lens_kept(want, off))


def lens_kept(keep, off):
    c = np.concatenate([[0], np.cumsum(keep, dtype=np.int64)])
    return c[off[1:]] - c[off[:-1]]


def _tie_band_ok(gpu_keep, ref_keep, ref_blocks, G, cutoff_score):
    bad = np.flatnonzero(gpu_keep != ref_keep)
    return all(abs(ref_blocks[i // G] - cutoff_score) <= RTOL * abs(cutoff_score) for i in bad)


@pytest.mark.timeout(600)
def test_acceptance_c8_identical_selection_across_tp(up, port, checker):
    cfgd = dict(query_window_n=8, block_size_g=8, sink_count_a=8, top_p=0.9)
    cfg = up.ScoreConfig(**cfgd)
    heads = up.HeadLayout(8, 8, 8)
    shifted = []
    for trial in range(100):
        n = 16 + port.rng_bits(trial, 0x6338, 0) % 497
        q = port.rng_normal_array(trial, 0x64617461, n * 64, 0.7).reshape(n, 64)
        k = port.rng_normal_array(trial, 0x64617461, n * 64, 0.7, first=1000000).reshape(n, 64)
        qb = torch.from_numpy(q).to(torch.bfloat16)
        kb = torch.from_numpy(k).to(torch.bfloat16)
        cu = torch.tensor([0, n], dtype=torch.int32, device="cuda")
        qd, kd = qb.reshape(n, 8, 8).cuda(), kb.reshape(n, 8, 8).cuda()
        sels = []
        for tp in (1, 2, 4, 8):
            res = up.score_blocks_tp(qd, kd, cu, cfg, tp, heads=heads, check=True)
            sel = up.select_varlen(res.block_scores, res.cu_blocks, cu, cfg, check=True)
            sels.append((sel.keep[:n].cpu().numpy(), int(sel.cutoff_rank[0]), res.block_scores[:(n + 7) // 8].cpu().numpy()))
        base_keep, base_cut, base_blk = sels[0]
        for tp, (kp, ct, blk) in zip((2, 4, 8), sels[1:]):
            if not (np.array_equal(kp, base_keep) and ct == base_cut):
                shifted.append((trial, tp))
                # only a tie at the cutoff may move the decision
                order = np.argsort(-base_blk, kind="stable")
                assert _tie_band_ok(kp, base_keep, base_blk, 8, base_blk[order[base_cut - 1]]), (trial, tp)
        if checker is not None:  # vs the reference on the same bf16-exact inputs
            _, red = checker.sharded_allreduce(qb.float().numpy(), kb.float().numpy(), 8, 8, 1, **cfgd)
            np.testing.assert_allclose(base_blk, red, rtol=RTOL, atol=1e-7)
            rsel = checker.top_p_select(red, n, **cfgd)
            order = np.argsort(-red, kind="stable")
            assert _tie_band_ok(base_keep, rsel.keep_mask, red, 8, red[order[rsel.cutoff_rank - 1]]), trial
    # acceptance c8 itself: identical selections on all 100 inputs
    assert shifted == []
