"""Generate golden vectors for the hot path from the UNMODIFIED reference (oracle/_ref).

Run in the build container (where /root/reference exists and oracle/_ref is built):
    python tests/golden/make_golden.py
Writes tests/golden/golden.json.  Floats are stored as IEEE-754 hex bit patterns so the
fixtures are exact.  Inputs are regenerated deterministically from the recorded seeds with
the reference's own CounterRng (rng.cpp:10-40, restated in oracle/uniprefill_oracle.c), so
only outputs and small inputs are stored.

Cases mirror the reference's own tests:
  selection: test_selection.cpp:152-317 KATs + acceptance c3-style random vectors
             (acceptance_main.cpp:175-217): zeros, quantised ties, denormals, uniforms;
  scorer:    score_tokens on seeded q/k (test_importance.cpp style), MHA and GQA;
  tp:        sharded_block_scores + allreduce_scores for T in {1,2,4,8} (test_tp_sim.cpp);
  compact:   patch_metadata KATs (test_scheduler.cpp:154-203) and apply_drop
             (test_propagation.cpp:97-111) on seeded rows.
"""
from __future__ import annotations

import json
import os
import struct
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402


def fhex(a) -> list:
    return [struct.pack("<f", float(x)).hex() for x in np.asarray(a, np.float32).ravel()]


def rng_matrix(port, rows, cols, seed, stream, stddev):
    return port.rng_normal_array(seed, stream, rows * cols, stddev).reshape(rows, cols)


def selection_cases(ref, port):
    cases = []
    kats = [
        ([0.5, 0.3, 0.15, 0.05], 4, dict(query_window_n=1, block_size_g=1, sink_count_a=0, top_p=0.9)),
        ([0.9, 0.05, 0.04, 0.01], 4, dict(query_window_n=1, block_size_g=1, sink_count_a=0, top_p=1.0)),
        ([0.1] * 10, 10, dict(query_window_n=1, block_size_g=1, sink_count_a=0, top_p=0.99)),
        ([0.0] * 5, 5, dict(query_window_n=1, block_size_g=1, sink_count_a=0, top_p=0.5)),
        ([0.0001] * 7 + [1.0] + [0.0001] * 12, 20, dict(query_window_n=1, block_size_g=1, sink_count_a=0, top_p=0.9)),
        ([1.0] * 50, 50, dict(query_window_n=1, block_size_g=1, sink_count_a=0, top_p=0.99)),
    ]
    for s, n, cfg in kats:
        cases.append(("kat", np.asarray(s, np.float32), n, cfg))
    # c3-style random vectors, lengths log-uniform to 4096 (acceptance_main.cpp:175-217)
    key = 0x6333
    ctr = 0
    for trial in range(160):
        u = port.rng_uniform(31, key, ctr); ctr += 1
        n = max(1, int(2.0 ** (u * 12.0)))
        s = np.zeros(n, np.float32)
        for i in range(n):
            kind = port.rng_bits(31, key, ctr) % 5; ctr += 1
            if kind == 0:
                s[i] = 0.0
            elif kind == 1:
                s[i] = np.float32(int(port.rng_uniform(31, key, ctr) * 8.0) * 0.125); ctr += 1
            elif kind == 2:
                s[i] = np.float32(1.4e-45) * np.float32(1 + port.rng_bits(31, key, ctr) % 7); ctr += 1
            else:
                s[i] = np.float32(port.rng_uniform(31, key, ctr)); ctr += 1
        p = 1.0 if trial % 7 == 0 else float(np.float32(0.3 + 0.7 * port.rng_uniform(31, key, ctr)))
        ctr += 1
        cases.append(("c3", s, n, dict(query_window_n=1, block_size_g=1, sink_count_a=0, top_p=p)))
    # blocks with sinks and window (test_selection.cpp:290-317 style)
    for trial in range(40):
        n = 40 + int(port.rng_bits(24, 0x636F76, 2 * trial) % 400)
        nb = (n + 7) // 8
        s = np.array([port.rng_uniform(24, 0x636F77 + trial, g) * port.rng_uniform(24, 0x636F78 + trial, g)
                      for g in range(nb)], np.float32)
        cases.append(("forced", s, n, dict(query_window_n=8, block_size_g=8, sink_count_a=8, top_p=0.8)))
    out = []
    for kind, s, n, cfg in cases:
        sel = ref.top_p_select(s, n, **cfg)
        out.append({"kind": kind, "scores": fhex(s), "num_tokens": n, "cfg": cfg,
                    "retained": sel.retained_indices.tolist(), "cutoff_rank": sel.cutoff_rank,
                    "covered_mass": sel.covered_mass.hex(), "degenerate": sel.degenerate_keep_all})
    return out


def scorer_cases(ref, port):
    specs = [  # (N, H, Hkv, D, cfg, seed)
        (40, 8, 8, 8, dict(query_window_n=16, block_size_g=8, sink_count_a=8, top_p=0.9), 1),  # score_default.json
        (300, 4, 2, 32, dict(query_window_n=16, block_size_g=8, sink_count_a=8, top_p=0.9), 2),
        (700, 8, 2, 64, dict(query_window_n=128, block_size_g=64, sink_count_a=128, top_p=0.99), 3),
        (1100, 4, 1, 128, dict(query_window_n=128, block_size_g=64, sink_count_a=128, top_p=0.99), 4),
        (515, 4, 2, 128, dict(query_window_n=100, block_size_g=32, sink_count_a=16, top_p=0.95), 5),
    ]
    out = []
    for N, H, Hkv, D, cfg, seed in specs:
        q = rng_matrix(port, N, H * D, seed, 0x696D70, 0.7)
        k = rng_matrix(port, N, Hkv * D, seed, 0x696D71, 0.7)
        tok, blk, n_eff = ref.score_tokens(q, k, H, Hkv, **cfg)
        sel = ref.top_p_select(blk, N, **cfg)
        out.append({"N": N, "H": H, "Hkv": Hkv, "D": D, "cfg": cfg, "seed": seed, "stddev": 0.7,
                    "token_scores": fhex(tok), "block_scores": fhex(blk), "effective_n": n_eff,
                    "retained": sel.retained_indices.tolist(), "cutoff_rank": sel.cutoff_rank})
    return out


def tp_cases(ref, port):
    out = []
    cfg = dict(query_window_n=8, block_size_g=8, sink_count_a=4, top_p=0.9)
    for trial, N in enumerate((40, 77, 130)):
        q = rng_matrix(port, N, 64, 100 + trial, 0x7470, 0.6)
        k = rng_matrix(port, N, 64, 200 + trial, 0x7470, 0.6)
        per_t = {}
        for tp in (1, 2, 4, 8):
            shards, red = ref.sharded_allreduce(q, k, 8, 8, tp, **cfg)
            per_t[str(tp)] = {"shards": [fhex(s) for s in shards], "reduced": fhex(red)}
        out.append({"N": N, "H": 8, "D": 8, "seed_q": 100 + trial, "seed_k": 200 + trial, "cfg": cfg,
                    "stddev": 0.6, "tp": per_t})
    return out


def compact_cases(ref, port):
    out = []
    toks = rng_matrix(port, 16, 8, 30, 0x636D70, 1.0)
    for name, cu, keep, sel, dec in [
        ("keep_half_first", [0, 8, 16], [1, 0, 1, 0, 1, 0, 1, 0] + [1] * 8, [1, 0], None),
        ("none_selected", [0, 8, 16], [1] * 16, [0, 0], None),
        ("prefill_decode", [0, 8, 9], [1, 1, 1, 1, 0, 0, 0, 0, 1], [1, 0], [0, 1]),
    ]:
        T = cu[-1]
        t, cu_out = ref.patch_metadata(toks[:T], cu, keep, sel, dec)
        out.append({"name": name, "cu": cu, "keep": keep, "selected": sel, "is_decode": dec,
                    "tokens": fhex(toks[:T]), "cols": 8, "cu_out": cu_out.tolist(), "out": fhex(t)})
    states = rng_matrix(port, 8, 32, 2, 0x70726F70, 1.0)
    keep = [1, 1, 0, 0, 0, 0, 1, 1]
    s, pos = ref.apply_drop(states, keep)
    out.append({"name": "apply_drop_order", "rows": 8, "cols": 32, "keep": keep, "states": fhex(states),
                "out": fhex(s), "positions": pos.tolist()})
    return out


def main():
    if not oracle.ref_available():
        raise SystemExit("oracle/_ref is not built (make -C oracle)")
    ref, port = oracle.ref(), oracle.port()
    doc = {
        "generator": "tests/golden/make_golden.py (reference: /root/reference/proj/core via oracle/_ref)",
        "phi": {str(x): ref.phi_encode(x) for x in (0.0, -0.0, 1.0, -1.0, 2.5, -3.75, 1.4e-45)},
        "selection": selection_cases(ref, port),
        "scorer": scorer_cases(ref, port),
        "tp": tp_cases(ref, port),
        "compact": compact_cases(ref, port),
    }
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
    with open(path, "w") as f:
        json.dump(doc, f, separators=(",", ":"))
    print(path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
