"""CPU, world_size 2 over gloo: the multi-GPU host logic.

* TP head sharding (tp_sim.cpp:12-49): each rank scores its head slice (here with the CPU
  oracle standing in for the GPU scorer) and ``allreduce_block_scores`` combines the
  partials.  The deterministic mode must reproduce the reference's ascending-shard fp32
  sum bit for bit; the all-reduce mode must match within fp32 rounding; every rank must
  then make the same selection (acceptance c8, acceptance_main.cpp:445-478).
* request sharding: LPT partition covers every request exactly once and is balanced.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2605_06221_b200.distributed import allreduce_block_scores, head_slice, shard_requests
        orc = oracle.port()
        cfg = dict(query_window_n=8, block_size_g=8, sink_count_a=8, top_p=0.9)
        H, Hkv, D, N = 8, 4, 16, 130
        rng = np.random.default_rng(7)
        q = rng.standard_normal((N, H * D)).astype(np.float32)
        k = rng.standard_normal((N, Hkv * D)).astype(np.float32)
        (qb, qe), (kb, ke) = head_slice(H, Hkv, rank, world)
        _, part, _ = orc.score_tokens_heads(q, k, H, Hkv, qb, qe, want_tokens=False, **cfg)
        t = torch.from_numpy(part.copy())

        def oracle_reducer(shards):
            return torch.from_numpy(orc.allreduce_scores([s.numpy() for s in shards], list(range(len(shards)))))

        det = allreduce_block_scores(t.clone(), deterministic=True, reducer=oracle_reducer)
        fast = allreduce_block_scores(t.clone(), deterministic=False)
        sel = orc.top_p_select(det.numpy(), N, **cfg)
        mine, local_cu = shard_requests([0, 100, 350, 351, 900, 1000], rank, world)
        out[rank] = dict(det=det.numpy().copy(), fast=fast.numpy().copy(), keep=sel.keep_mask.copy(),
                         mine=mine, local_cu=local_cu)
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def results():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    return dict(out)


def test_tp_deterministic_reduction_matches_reference(results):
    import oracle
    port = oracle.port()
    cfg = dict(query_window_n=8, block_size_g=8, sink_count_a=8, top_p=0.9)
    rng = np.random.default_rng(7)
    H, Hkv, D, N = 8, 4, 16, 130
    q = rng.standard_normal((N, H * D)).astype(np.float32)
    k = rng.standard_normal((N, Hkv * D)).astype(np.float32)
    shards = [port.score_tokens_heads(q, k, H, Hkv, t * 4, (t + 1) * 4, want_tokens=False, **cfg)[1]
              for t in range(2)]
    want = port.allreduce_scores(shards, [0, 1])
    for r in (0, 1):
        assert np.array_equal(results[r]["det"], want)
        np.testing.assert_allclose(results[r]["fast"], want, rtol=1e-6)
    if oracle.ref_available():
        _, red = oracle.ref().sharded_allreduce(q, k, H, Hkv, 2, **cfg)
        assert np.array_equal(want, red)


def test_tp_ranks_select_identically(results):
    assert np.array_equal(results[0]["keep"], results[1]["keep"])


def test_request_sharding_partition(results):
    mine = sorted(results[0]["mine"] + results[1]["mine"])
    assert mine == list(range(5))
    lengths = [100, 250, 1, 549, 100]
    loads = [sum(lengths[i] for i in results[r]["mine"]) for r in (0, 1)]
    assert max(loads) - min(loads) <= max(lengths)
    for r in (0, 1):
        cu = results[r]["local_cu"]
        assert cu[0] == 0 and cu[-1] == loads[r]


def test_head_slice_replicates_kv_heads_for_qwen_tp8():
    from paper_2605_06221_b200.distributed import head_slice
    # Qwen3-Next FA layer: Hq=16, Hkv=2, TP=8 -> 2 q-heads per rank, one kv-head each.
    slices = [head_slice(16, 2, t, 8) for t in range(8)]
    assert [s[0] for s in slices] == [(2 * t, 2 * t + 2) for t in range(8)]
    assert [s[1] for s in slices] == [(0, 1)] * 4 + [(1, 2)] * 4
