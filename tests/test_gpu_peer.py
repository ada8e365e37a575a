"""GPU: the TP score all-reduce over peer memory (up_peer_allreduce_scores,
distributed.PeerScoreReducer) against allreduce_scores' ascending-rank fp32 sum
(tp_sim.cpp:43-47), bit for bit.

The GPU pool gives one GPU per call, so the TP group here is two processes sharing cuda:0:
the exchange buffers are mapped across the processes with CUDA IPC exactly as across GPUs
(the kernels of the two processes time-slice on the device, so this checks the protocol --
stores, flags, epochs, graph replay -- not NVLink speed)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

COUNTS = [1, 300, 8192, 40000, 777]


def _partial(rank, step, n):
    g = torch.Generator().manual_seed(1000 * step + rank)
    return torch.rand(n, generator=g, dtype=torch.float64).mul(10).float()


def _expected(tp, step, n):
    acc = np.zeros(n, dtype=np.float32)
    for t in range(tp):  # ((0.0f + s_0) + s_1) + ... in fp32
        acc = (acc + _partial(t, step, n).numpy()).astype(np.float32)
    return acc


def _worker(rank, tp, port, q):
    import torch.distributed as dist
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=tp)
        from paper_2605_06221_b200.distributed import PeerScoreReducer, allreduce_block_scores
        red = PeerScoreReducer(max(COUNTS), device="cuda:0")
        bad = []
        for step, n in enumerate(COUNTS):
            part = _partial(rank, step, n).cuda()
            out = torch.empty_like(part)
            red(part, out)
            if step % 2:  # in place through the allreduce_block_scores entry point
                allreduce_block_scores(part, peer=red)
                if not torch.equal(part, out):
                    bad.append(f"in-place step {step}")
            torch.cuda.synchronize()
            red.check()
            if not np.array_equal(out.cpu().numpy().view(np.uint32), _expected(tp, step, n).view(np.uint32)):
                bad.append(f"step {step} n={n}")
        # CUDA graph: the rendezvous state (flags, epoch) lives on the device
        n = 5000
        part = torch.empty(n, device="cuda:0")
        out = torch.empty_like(part)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            part.copy_(_partial(rank, 50, n))
            red(part, out)  # warm-up outside capture
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                red(part, out)
        torch.cuda.synchronize()
        dist.barrier()
        for step in (51, 52):
            part.copy_(_partial(rank, step, n))
            torch.cuda.synchronize()
            g.replay()
            torch.cuda.synchronize()
            if not np.array_equal(out.cpu().numpy().view(np.uint32), _expected(tp, step, n).view(np.uint32)):
                bad.append(f"graph replay {step}")
        red.check()
        # back-to-back stress, no host sync between calls (the write-after-read window of a
        # single-bank exchange): STRESS calls with different data and counts, eager and then
        # captured in one graph, every output checked bitwise afterwards.
        STRESS = 128
        ns = [1 + (37 * i) % 6000 for i in range(STRESS)]
        parts = [_partial(rank, 100 + i, n).cuda() for i, n in enumerate(ns)]
        outs = [torch.full_like(pt, float("nan")) for pt in parts]
        want = [_expected(tp, 100 + i, n).view(np.uint32) for i, n in enumerate(ns)]
        torch.cuda.synchronize()
        dist.barrier()
        with torch.cuda.stream(s):
            for pt, o in zip(parts, outs):
                red(pt, o)
        torch.cuda.synchronize()
        red.check()
        bad += [f"stress eager call {i}" for i in range(STRESS)
                if not np.array_equal(outs[i].cpu().numpy().view(np.uint32), want[i])]
        for o in outs:
            o.fill_(float("nan"))
        torch.cuda.synchronize()
        with torch.cuda.stream(s):
            g2 = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g2, stream=s):
                for pt, o in zip(parts[:64], outs[:64]):
                    red(pt, o)
        torch.cuda.synchronize()
        dist.barrier()
        for rep in range(3):
            g2.replay()  # replays back to back, no sync in between
        torch.cuda.synchronize()
        red.check()
        bad += [f"stress graph call {i}" for i in range(64)
                if not np.array_equal(outs[i].cpu().numpy().view(np.uint32), want[i])]
        red.close()
        dist.destroy_process_group()
        q.put((rank, bad))
    except Exception:  # report instead of hanging the parent
        import traceback
        tb = traceback.format_exc()
        os.makedirs("gpurun_out", exist_ok=True)
        with open(f"gpurun_out/peer_rank{rank}.txt", "w") as f:
            f.write(tb)
        q.put((rank, [tb.strip().splitlines()[-1]]))


@pytest.mark.timeout(300)
@pytest.mark.parametrize("tp", [2, 3])
def test_peer_allreduce_bitwise_ranks_one_device(tp):
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, tp, port, q)) for r in range(tp)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=250) for _ in procs)
    for p in procs:
        p.join(timeout=30)
    assert results == {r: [] for r in range(tp)}, results


def _worker_fused(rank, tp, port, q):
    import torch.distributed as dist
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=tp)
        import paper_2605_06221_b200 as up
        from paper_2605_06221_b200.distributed import PeerScoreReducer, head_slice
        from paper_2605_06221_b200.synthetic import make_batch
        bad = []
        for case, (lengths, Hq, Hkv, D) in enumerate([([3000, 1500, 64], 8, 2, 128),     # GQA-4, HPC 4 slices
                                                      ([5000], 4, 4, 256),             # MHA, D=256
                                                      ([700, 2100], 8, 1, 64)]):       # kv-head shared by ranks
            sb = make_batch(lengths, Hq, Hkv, D, 64, regime="planted", seed=7 + case, device="cuda:0")
            cfg = up.ScoreConfig()
            nb = sum((n + 63) // 64 for n in lengths)
            red = PeerScoreReducer(nb + len(lengths) + 1, device="cuda:0")
            slices = [head_slice(Hq, Hkv, t, tp) for t in range(tp)]

            def layout(t):
                (qb, qe), (kb, ke) = slices[t]
                return up.HeadLayout(qe - qb, ke - kb, D, gqa_group=Hq // Hkv, q_head_offset=qb, kv_head_offset=kb)

            (qb, qe), (kb, ke) = slices[rank]
            ws = up.Workspace("cuda:0")
            for rep in range(3):  # repeated calls: flags / epochs advance
                got = red.score_blocks(sb.q[:, qb:qe], sb.k[:, kb:ke], sb.cu_seqlens, cfg, layout(rank),
                                       workspace=ws)
                torch.cuda.synchronize()
                ws.device_status()
            # the same partials through the plain scorer, summed in ascending rank order
            parts = []
            for t in range(tp):
                (tqb, tqe), (tkb, tke) = slices[t]
                parts.append(up.score_blocks_varlen(sb.q[:, tqb:tqe], sb.k[:, tkb:tke], sb.cu_seqlens, cfg,
                                                    layout(t)).block_scores[:nb].cpu().numpy())
            want = np.zeros(nb, dtype=np.float32)
            for t in range(tp):
                want = (want + parts[t]).astype(np.float32)
            if not np.array_equal(got.block_scores[:nb].cpu().numpy().view(np.uint32), want.view(np.uint32)):
                bad.append(f"case {case}: fused != ascending sum of the partials")
            red.close()
        dist.destroy_process_group()
        q.put((rank, bad))
    except Exception:
        import traceback
        q.put((rank, [traceback.format_exc().strip().splitlines()[-1]]))


@pytest.mark.timeout(300)
def test_fused_score_and_peer_allreduce_two_ranks_one_device():
    """up_score_blocks_peer: each rank's head slice scored, the combine kernel storing its
    partials straight into the peers, bitwise the ascending-rank sum of the per-rank
    partials of the plain scorer."""
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker_fused, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=280) for _ in procs)
    for p in procs:
        p.join(timeout=30)
    assert results == {0: [], 1: []}, results
