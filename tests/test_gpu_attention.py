"""GPU parity: the drop layer's attention readout over the retained rows
(up_attention_varlen) against the unmodified reference's
attention_readout (model.cpp:215-263, through oracle/_ref) on the same bf16-rounded inputs,
and at larger sizes against a plain PyTorch fp32 restatement.

Tolerance: P is rounded to bf16 before the P·V MMA and the output is bf16, so every output
element is within 2e-2 * (1 + |ref|) of the fp32/fp64 reference (bf16 carries 8 bits)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

TOL = 2e-2


def _inputs(lengths, Hq, Hkv, D, seed, gap=3):
    g = torch.Generator().manual_seed(seed)
    T = sum(lengths)
    q = torch.randn(T, Hq, D, generator=g).to(torch.bfloat16)
    k = torch.randn(T, Hkv, D, generator=g).to(torch.bfloat16)
    v = torch.randn(T, Hkv, D, generator=g).to(torch.bfloat16)
    pos = []
    for n in lengths:  # retained logical positions: strictly increasing with random gaps
        steps = torch.randint(1, gap + 1, (n,), generator=g)
        pos.append(torch.cumsum(steps, 0) - 1)
    pos = torch.cat(pos).to(torch.int64)
    cu = torch.tensor(np.concatenate([[0], np.cumsum(lengths)]), dtype=torch.int32)
    return q, k, v, pos, cu


def _torch_ref(q, k, v, pos, cu, window=0):
    """fp32 restatement of attention_readout per segment (GQA by head // group)."""
    T, Hq, D = q.shape
    group = Hq // k.shape[1]
    out = torch.zeros(T, Hq, D, dtype=torch.float32, device=q.device)
    qf, kf, vf = q.float(), k.float().repeat_interleave(group, 1), v.float().repeat_interleave(group, 1)
    for r in range(cu.numel() - 1):
        b, e = int(cu[r]), int(cu[r + 1])
        p = pos[b:e]
        vis = p[None, :] <= p[:, None]
        if window > 0:
            vis &= p[None, :] > p[:, None] - window
        for c0 in range(b, e, 2048):
            c1 = min(c0 + 2048, e)
            s = torch.einsum("ihd,jhd->hij", qf[c0:c1], kf[b:e]) / D ** 0.5
            s = s.masked_fill(~vis[c0 - b:c1 - b][None], float("-inf"))
            out[c0:c1] = torch.einsum("hij,jhd->ihd", torch.softmax(s, -1), vf[b:e])
    return out


def _close(got, want):
    err = (got.float() - want).abs()
    bad = err > TOL * (1 + want.abs())
    assert not bool(bad.any()), f"{int(bad.sum())} elements off, max err {float(err.max()):.4g}"


@pytest.mark.parametrize("lengths,Hq,Hkv,D,window", [
    ([300], 4, 2, 128, 0),
    ([1, 129, 257, 64], 4, 1, 128, 0),
    ([500, 70], 2, 2, 64, 0),
    ([400], 4, 2, 128, 40),
    ([256, 130], 8, 2, 64, 200),
    ([300, 65, 1], 4, 2, 256, 0),
    ([200], 2, 1, 256, 50),
])
def test_attention_matches_reference(up, ref, lengths, Hq, Hkv, D, window):
    q, k, v, pos, cu = _inputs(lengths, Hq, Hkv, D, seed=sum(lengths) + D + window)
    got = up.attention_varlen(q.cuda(), k.cuda(), v.cuda(), cu.cuda(), pos.cuda(), window=window, check=True)
    got = got.cpu()
    for r in range(len(lengths)):
        b, e = int(cu[r]), int(cu[r + 1])
        want = ref.attention_readout(q[b:e].float().reshape(e - b, -1).numpy(), pos[b:e].numpy(),
                                     k[b:e].float().reshape(e - b, -1).numpy(),
                                     v[b:e].float().reshape(e - b, -1).numpy(), pos[b:e].numpy(), Hq, Hkv, window)
        _close(got[b:e].reshape(e - b, -1), torch.from_numpy(want))


@pytest.mark.parametrize("lengths,Hq,Hkv,D,window", [
    ([8192], 32, 8, 128, 0),
    ([3000, 5000, 1, 777], 8, 8, 128, 0),
    ([6000, 2048], 16, 4, 64, 1024),
    ([4096, 1000], 16, 2, 256, 0),     # Qwen3-Next full-attention head layout
    ([3000, 64], 16, 8, 256, 1024),    # Gemma-3 head layout, sliding window
])
def test_attention_large_vs_torch(up, lengths, Hq, Hkv, D, window):
    q, k, v, pos, cu = _inputs(lengths, Hq, Hkv, D, seed=7 + D)
    q, k, v, pos, cu = q.cuda(), k.cuda(), v.cuda(), pos.cuda(), cu.cuda()
    got = up.attention_varlen(q, k, v, cu, pos, window=window, check=True)
    _close(got, _torch_ref(q, k, v, pos, cu.cpu(), window))


def test_attention_after_drop_layer(up):
    """The drop layer end to end: score -> select -> compact the q/k/v/position planes, then
    attention over the retained rows equals the reference readout over the gathered rows."""
    from paper_2605_06221_b200.synthetic import make_batch
    lengths = [4096, 1500]
    Hq, Hkv, D = 32, 8, 128
    sb = make_batch(lengths, Hq, Hkv, D, 64, regime="planted", seed=5, device="cuda")
    T = sum(lengths)
    layer = up.DropLayer(up.ScoreConfig(), up.HeadLayout(Hq, Hkv, D), T, len(lengths),
                         [(Hq, D), (Hkv, D), (Hkv, D), ()], [torch.bfloat16] * 3 + [torch.int64])
    res = layer(sb.q, sb.k, sb.cu_seqlens, [sb.q, sb.k, sb.v, sb.positions])
    layer.check()
    n = int(res.num_out.item())
    assert n < T  # something was dropped
    qc, kc, vc, pc = res.planes
    got = up.attention_varlen(qc, kc, vc, res.cu_seqlens, pc, max_tokens=T, check=True)[:n]
    keep = layer.sel.keep.bool()
    want = _torch_ref(sb.q[keep], sb.k[keep], sb.v[keep], sb.positions[keep], res.cu_seqlens.cpu())
    _close(got, want)


def test_attention_cuda_graph_and_launch_count(up):
    q, k, v, pos, cu = _inputs([1000, 24], 4, 2, 128, seed=1)
    q, k, v, pos, cu = q.cuda(), k.cuda(), v.cuda(), pos.cuda(), cu.cuda()
    out = torch.zeros_like(q)
    eager = up.attention_varlen(q, k, v, cu, pos).clone()
    assert up.lib.up_last_launch_count() == 1
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        up.attention_varlen(q, k, v, cu, pos, out=out)  # warm
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            up.attention_varlen(q, k, v, cu, pos, out=out)
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, eager)


@pytest.mark.parametrize("D,Hq,Hkv", [(128, 8, 2), (256, 4, 2)])
def test_attention_ignores_garbage_past_the_batch(up, D, Hq, Hkv):
    """Capacity-sized buffers: rows past cu_seqlens[-1] hold NaN (an uninitialised compaction
    output).  Masked keys must contribute exactly nothing -- no 0 * NaN from the PV MMA."""
    lengths = [300, 77]
    q, k, v, pos, cu = _inputs(lengths, Hq, Hkv, D, seed=31)
    n, cap = sum(lengths), 1000
    def padded(x):
        y = torch.full((cap,) + tuple(x.shape[1:]), float("nan"), dtype=x.dtype)
        y[:n] = x
        return y.cuda()
    qp, kp, vp = padded(q), padded(k), padded(v)
    pp = torch.zeros(cap, dtype=torch.int64)
    pp[:n] = pos
    got = up.attention_varlen(qp, kp, vp, cu.cuda(), pp.cuda(), max_tokens=cap, check=True)[:n]
    assert bool(torch.isfinite(got.float()).all())
    _close(got, _torch_ref(q.cuda(), k.cuda(), v.cuda(), pos.cuda(), cu, 0))
