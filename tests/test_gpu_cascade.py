"""GPU: the cascaded drop path as the reference runs it -- stacked drops inside a block act
on the already-compacted stream, and the block boundary reconstitutes the full stream
(propagation.cpp:240-290, scheduler.cpp:283-361; stacked-drops oracle
test_propagation.cpp:113-143).

Two DropLayers in sequence: drop 1 scores, selects and compacts the batch; drop 2 scores
the stream drop 1 compacted -- its q/k rows are the compacted rows, its batch is drop 1's
DEVICE-resident cu_seqlens_out under the same capacity-sized launches -- then the block
boundary unwinds drop 2 and drop 1 (up_scatter_rows).  Checked per request against the
oracle: each drop's block scores within rtol 1e-3 and keep masks equal outside the tie band
(rule 2), the composed survivors = composition of the two masks over logical positions,
and the reconstituted stream = the pre-drop rows with the retained rows' new states.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

RTOL = 1e-3
CFG = dict(query_window_n=128, block_size_g=64, sink_count_a=128, top_p=0.99)


def _tie_band(keep, want_keep, ref_blk, G, cutoff):
    bad_blocks = {i // G for i in np.flatnonzero(keep != want_keep)}
    return all(abs(ref_blk[g] - cutoff) <= RTOL * abs(cutoff) for g in bad_blocks)


def _check_drop(port, q, k, cu, bs, cub, keep, Hq, Hkv):
    for r in range(len(cu) - 1):
        s, e = int(cu[r]), int(cu[r + 1])
        qq = q[s:e].float().reshape(e - s, -1).cpu().numpy()
        kk = k[s:e].float().reshape(e - s, -1).cpu().numpy()
        _, ref_blk, _ = port.score_tokens(qq, kk, Hq, Hkv, want_tokens=False, **CFG)
        got = bs[cub[r]:cub[r + 1]]
        np.testing.assert_allclose(got, ref_blk, rtol=RTOL, atol=1e-6 * ref_blk.sum() / len(ref_blk))
        ref_sel = port.top_p_select(ref_blk, e - s, **CFG)
        order = np.argsort(-ref_blk, kind="stable")
        cutoff = ref_blk[order[ref_sel.cutoff_rank - 1]]
        assert _tie_band(keep[s:e], ref_sel.keep_mask, ref_blk, CFG["block_size_g"], cutoff), f"request {r}"
        assert np.array_equal(keep[s:e], port.top_p_select(got, e - s, **CFG).keep_mask)  # rule 1


@pytest.mark.parametrize("lengths", [[3000, 1500, 700], [4096, 65, 2500, 1]])
def test_two_cascaded_drops_and_reconstitution(up, port, lengths):
    from paper_2605_06221_b200.synthetic import make_batch
    Hq, Hkv, D, HID = 8, 2, 128, 64
    R, T = len(lengths), sum(lengths)
    heads = up.HeadLayout(Hq, Hkv, D)
    cfg = up.ScoreConfig(**CFG)
    shapes, dtypes = [(HID,), (Hkv, D), (Hkv, D), ()], [torch.bfloat16, torch.bfloat16, torch.bfloat16, torch.int64]
    sb1 = make_batch(lengths, Hq, Hkv, D, HID, regime="planted", seed=sum(lengths) + 1)
    sb2 = make_batch(lengths, Hq, Hkv, D, HID, regime="planted", seed=sum(lengths) + 2)  # drop 2's q/k/v rows
    L1 = up.DropLayer(cfg, heads, T, R, shapes, dtypes)
    L2 = up.DropLayer(cfg, heads, T, R, shapes, dtypes)
    resid = sb1.hidden.clone()
    o1 = L1(sb1.q, sb1.k, sb1.cu_seqlens, [resid, sb1.k, sb1.v, sb1.positions])
    # drop 2 on the compacted stream: device cu_seqlens_out, capacity-sized launches
    o2 = L2(sb2.q, sb2.k, o1.cu_seqlens, [o1.planes[0], sb2.k, sb2.v, o1.planes[3]])
    L1.check()
    L2.check()
    n1, n2 = int(o1.num_out.item()), int(o2.num_out.item())
    cu1 = sb1.cu_seqlens.cpu().numpy()
    cu2 = o1.cu_seqlens.cpu().numpy()
    keep1 = L1.sel.keep.cpu().numpy()
    keep2 = L2.sel.keep.cpu().numpy()
    _check_drop(port, sb1.q, sb1.k, cu1, L1.scores.block_scores.cpu().numpy(), L1.scores.cu_blocks.cpu().numpy(),
                keep1, Hq, Hkv)
    # drop 2 saw exactly drop 1's compacted segments: its rows are sb2's first n1 rows
    _check_drop(port, sb2.q, sb2.k, cu2, L2.scores.block_scores.cpu().numpy(), L2.scores.cu_blocks.cpu().numpy(),
                keep2, Hq, Hkv)
    assert int(cu2[-1]) == n1
    # composition over logical positions (test_propagation.cpp:113-143)
    first = np.flatnonzero(keep1[:T])
    survivors = first[np.flatnonzero(keep2[:n1])]
    assert np.array_equal(o2.planes[3][:n2].cpu().numpy(), sb1.positions.cpu().numpy()[survivors])
    assert np.array_equal(o2.planes[0][:n2].view(torch.int16).cpu().numpy(),
                          sb1.hidden.view(torch.int16).cpu().numpy()[survivors])
    # the sublayers after drop 2 transform the retained rows; the block boundary unwinds
    new_state = torch.randn(n2, HID, device="cuda").to(torch.bfloat16)
    o2.planes[0][:n2] = new_state
    up.reconstitute_varlen([o2.planes[0]], o2, [o1.planes[0]])  # drop 2 -> drop-1 row space
    up.reconstitute_varlen([o1.planes[0]], o1, [resid])         # drop 1 -> the full stream
    want = sb1.hidden.clone()
    want[torch.from_numpy(survivors).cuda().long()] = new_state
    assert torch.equal(resid, want)
