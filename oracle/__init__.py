"""CPU oracle for the UniPrefill token-selection hot path -- TEST INFRASTRUCTURE ONLY.

Two checkers live here, both reached through ctypes:

* ``port``: the plain-C restatement in ``uniprefill_oracle.c`` (each function cites the
  reference file:line it restates), built to ``_build/liboracle_port.so``;
* ``ref``: the unmodified reference core compiled from ``/root/reference/proj/core/src``
  plus ``ref_shim.cpp`` into ``_ref/libuniprefill_ref.so`` (absent on machines where it
  was never built; the GPU box receives the prebuilt file with the repo snapshot).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this package, and only as the checker or the timed
CPU baseline -- never on the product path (``paper_2605_06221_b200``), which has no CPU
fallback.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "liboracle_port.so")
REF_SO = os.path.join(HERE, "_ref", "libuniprefill_ref.so")

OK, ERR_CONFIG, ERR_CONTRACT, ERR_ALLOCATION_MISS = 0, 1, 2, 3


class OracleConfigError(Exception):
    """Reference ConfigError (errors.hpp:15-18)."""


class OracleContractViolation(Exception):
    """Reference ContractViolation (errors.hpp:22-25)."""


class OracleAllocationMiss(Exception):
    """Reference AllocationMissError (errors.hpp:32-35)."""


def _raise(status: int, what: str) -> None:
    if status == OK:
        return
    if status == ERR_CONFIG:
        raise OracleConfigError(what)
    if status == ERR_CONTRACT:
        raise OracleContractViolation(what)
    if status == ERR_ALLOCATION_MISS:
        raise OracleAllocationMiss(what)
    raise RuntimeError(f"{what}: oracle status {status}")


class _ModelCfg(ctypes.Structure):
    _fields_ = [("num_blocks", ctypes.c_int32), ("sublayers_per_block", ctypes.c_int32),
                ("hidden_dim", ctypes.c_int32), ("head_dim", ctypes.c_int32), ("num_heads", ctypes.c_int32),
                ("window_size", ctypes.c_int32), ("ffn_dim", ctypes.c_int32),
                ("layer_pattern", ctypes.POINTER(ctypes.c_int32))]


def _model_cfg(cfg):
    """ctypes view of a paper_2605_06221_b200.ledger.ModelConfig (keeps the pattern alive)."""
    pat = np.ascontiguousarray([int(k) for k in cfg.layer_pattern], dtype=np.int32)
    c = _ModelCfg(cfg.num_blocks, cfg.sublayers_per_block, cfg.hidden_dim, cfg.head_dim, cfg.num_heads,
                  cfg.window_size, cfg.ffn_dim, _ptr(pat, ctypes.c_int32))
    return c, pat


class _Cfg(ctypes.Structure):
    _fields_ = [("query_window_n", ctypes.c_int32), ("block_size_g", ctypes.c_int32),
                ("sink_count_a", ctypes.c_int32), ("top_p", ctypes.c_float)]


class _SelInfo(ctypes.Structure):
    _fields_ = [("cutoff_rank", ctypes.c_int64), ("retained_count", ctypes.c_int64),
                ("retention_ratio", ctypes.c_double), ("covered_mass", ctypes.c_double),
                ("degenerate_keep_all", ctypes.c_int32)]


@dataclass
class OracleSelection:
    keep_mask: np.ndarray
    cutoff_rank: int
    retained_count: int
    retention_ratio: float
    covered_mass: float
    degenerate_keep_all: bool

    @property
    def retained_indices(self) -> np.ndarray:
        return np.flatnonzero(self.keep_mask).astype(np.int64)


def build() -> None:
    """Compile the port (and, when the reference sources are present, the reference)."""
    subprocess.run(["make", "-s", "-C", HERE, "-j8"], check=True)


def _ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(ctypes.POINTER(ctype))


def _cfg(query_window_n=128, block_size_g=64, sink_count_a=128, top_p=0.99) -> _Cfg:
    return _Cfg(int(query_window_n), int(block_size_g), int(sink_count_a), float(top_p))


class _Lib:
    """Common ctypes surface of the port (orc_*) and the reference shim (ref_*)."""

    def __init__(self, path: str, prefix: str):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.path = path
        self.lib = ctypes.CDLL(path)
        self.prefix = prefix
        f = self._fn
        P = ctypes.POINTER
        f("phi_encode", [ctypes.c_float, P(ctypes.c_uint32)])
        f("phi_decode", [ctypes.c_uint32], ctypes.c_float)
        f("score_tokens_heads", [P(ctypes.c_float), ctypes.c_int64, P(ctypes.c_float), ctypes.c_int64,
                                 ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                 ctypes.c_int, P(_Cfg), P(ctypes.c_float), P(ctypes.c_float),
                                 P(ctypes.c_int32)])
        f("top_p_select", [P(ctypes.c_float), ctypes.c_int64, P(_Cfg), ctypes.c_int64,
                           P(ctypes.c_uint8), P(_SelInfo)])
        f("expand_mask", [P(ctypes.c_uint8), ctypes.c_int64, ctypes.c_int, ctypes.c_int64,
                          ctypes.c_int64, ctypes.c_int64, P(ctypes.c_uint8)])
        f("allreduce_scores", [P(P(ctypes.c_float)), P(ctypes.c_int32), ctypes.c_int32,
                               ctypes.c_int64, P(ctypes.c_float)])

    def _fn(self, name, argtypes, restype=ctypes.c_int):
        fn = getattr(self.lib, f"{self.prefix}_{name}")
        fn.argtypes = argtypes
        fn.restype = restype
        return fn

    def _call(self, name):
        return getattr(self.lib, f"{self.prefix}_{name}")

    # ---- phi -------------------------------------------------------------
    def phi_encode(self, x: float) -> int:
        out = ctypes.c_uint32(0)
        _raise(self._call("phi_encode")(ctypes.c_float(x), ctypes.byref(out)), "phi_encode")
        return int(out.value)

    def phi_decode(self, bits: int) -> float:
        return float(self._call("phi_decode")(ctypes.c_uint32(bits)))

    # ---- scorer ----------------------------------------------------------
    def score_tokens_heads(self, q: np.ndarray, k: np.ndarray, num_heads: int, num_kv_heads: int,
                           head_begin: int, head_end: int, want_tokens: bool = True, **cfg):
        """q: N x (H*D), k: N x (Hkv*D) float32.  Returns (token_scores, block_scores, n_eff)."""
        q = np.ascontiguousarray(q, dtype=np.float32)
        k = np.ascontiguousarray(k, dtype=np.float32)
        N = q.shape[0]
        D = q.shape[1] // num_heads
        c = _cfg(**cfg)
        G = c.block_size_g
        nb = (N + G - 1) // G if G > 0 else 0
        tok = np.zeros(max(N, 1), np.float32)
        blk = np.zeros(max(nb, 1), np.float32)
        n_eff = ctypes.c_int32(0)
        st = self._call("score_tokens_heads")(
            _ptr(q, ctypes.c_float), q.shape[1], _ptr(k, ctypes.c_float), k.shape[1], N, num_heads,
            num_kv_heads, D, head_begin, head_end, ctypes.byref(c),
            _ptr(tok, ctypes.c_float) if want_tokens else None, _ptr(blk, ctypes.c_float),
            ctypes.byref(n_eff))
        _raise(st, "score_tokens_heads")
        return tok[:N], blk[:nb], int(n_eff.value)

    def score_tokens(self, q, k, num_heads, num_kv_heads=None, **cfg):
        kvh = num_heads if num_kv_heads is None else num_kv_heads
        return self.score_tokens_heads(q, k, num_heads, kvh, 0, num_heads, **cfg)

    # ---- selection -------------------------------------------------------
    def top_p_select(self, block_scores, num_tokens: int, **cfg) -> OracleSelection:
        b = np.ascontiguousarray(block_scores, dtype=np.float32)
        keep = np.zeros(max(num_tokens, 1), np.uint8)
        info = _SelInfo()
        c = _cfg(**cfg)
        st = self._call("top_p_select")(_ptr(b, ctypes.c_float), b.size, ctypes.byref(c), num_tokens,
                                        _ptr(keep, ctypes.c_uint8), ctypes.byref(info))
        _raise(st, "top_p_select")
        return OracleSelection(keep[:num_tokens].copy(), info.cutoff_rank, info.retained_count,
                               info.retention_ratio, info.covered_mass,
                               bool(info.degenerate_keep_all))

    def expand_mask(self, block_mask, block_size, num_tokens, sink_count, window_n) -> np.ndarray:
        bm = np.ascontiguousarray(block_mask, dtype=np.uint8)
        keep = np.zeros(max(num_tokens, 1), np.uint8)
        st = self._call("expand_mask")(_ptr(bm, ctypes.c_uint8), bm.size, block_size, num_tokens,
                                       sink_count, window_n, _ptr(keep, ctypes.c_uint8))
        _raise(st, "expand_mask")
        return keep[:num_tokens]

    def allreduce_scores(self, shards, shard_ids) -> np.ndarray:
        arrs = [np.ascontiguousarray(s, dtype=np.float32) for s in shards]
        length = arrs[0].size if arrs else 0
        ptrs = (ctypes.POINTER(ctypes.c_float) * max(len(arrs), 1))(*[_ptr(a, ctypes.c_float) for a in arrs])
        ids = np.ascontiguousarray(shard_ids, dtype=np.int32)
        out = np.zeros(max(length, 1), np.float32)
        st = self._call("allreduce_scores")(ptrs, _ptr(ids, ctypes.c_int32), len(arrs), length,
                                            _ptr(out, ctypes.c_float))
        _raise(st, "allreduce_scores")
        return out[:length]


class Port(_Lib):
    """The C restatement (uniprefill_oracle.c)."""

    def __init__(self, path: str = PORT_SO):
        super().__init__(path, "orc")
        P = ctypes.POINTER
        self._fn("restrict_selection", [P(ctypes.c_uint8), P(ctypes.c_uint8), ctypes.c_int64,
                                        P(ctypes.c_float), ctypes.c_int64, ctypes.c_int, P(_SelInfo)])
        self._fn("compact", [P(ctypes.c_uint8), P(ctypes.c_int64), ctypes.c_int32, P(ctypes.c_uint8),
                             ctypes.c_int32, P(ctypes.c_void_p), P(ctypes.c_void_p), P(ctypes.c_int64),
                             P(ctypes.c_int64), P(ctypes.c_int64), P(ctypes.c_int64)])
        self._fn("rng_key", [ctypes.c_uint64, ctypes.c_uint64], ctypes.c_uint64)
        self._fn("rng_bits", [ctypes.c_uint64, ctypes.c_uint64], ctypes.c_uint64)
        self._fn("rng_uniform", [ctypes.c_uint64, ctypes.c_uint64], ctypes.c_double)
        self._fn("rng_normal", [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_double], ctypes.c_float)
        self._fn("scoring_flops", [ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_int],
                 ctypes.c_uint64)
        self._fn("reconstitute", [ctypes.c_void_p, P(ctypes.c_int64), ctypes.c_int64, ctypes.c_void_p,
                                  P(ctypes.c_int64), ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                  ctypes.c_void_p])
        self._fn("slot_for", [P(ctypes.c_int64), ctypes.c_int64, ctypes.c_int, ctypes.c_int64, P(ctypes.c_int64)])
        self._fn("decode_seqused", [ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, P(ctypes.c_int32),
                                    P(ctypes.c_int64), ctypes.c_int32], ctypes.c_int64)

    def reconstitute(self, active: np.ndarray, active_pos, parked: np.ndarray, parked_pos) -> np.ndarray:
        """reconstitute (propagation.cpp:79-100) of one stream."""
        a = np.ascontiguousarray(active)
        pk = np.ascontiguousarray(parked, dtype=a.dtype).reshape(-1, *a.shape[1:])
        ap = np.ascontiguousarray(active_pos, dtype=np.int64)
        pp = np.ascontiguousarray(parked_pos, dtype=np.int64)
        n = ap.size + pp.size
        out = np.zeros((n, *a.shape[1:]), a.dtype)
        rb = a[0].nbytes if a.shape[0] else pk[0].nbytes
        st = self.lib.orc_reconstitute(a.ctypes.data, _ptr(ap, ctypes.c_int64), ap.size, pk.ctypes.data,
                                       _ptr(pp, ctypes.c_int64), pp.size, rb, n, out.ctypes.data)
        _raise(st, "reconstitute")
        return out

    def slot_for(self, table, block_size: int, pos: int) -> int:
        t = np.ascontiguousarray(table, dtype=np.int64)
        out = ctypes.c_int64(0)
        _raise(self.lib.orc_slot_for(_ptr(t, ctypes.c_int64), t.size, block_size, pos, ctypes.byref(out)),
               "slot_for")
        return int(out.value)

    def decode_seqused(self, original_length: int, decode_appended: int, event_layers, retained_lengths,
                       layer: int) -> int:
        el = np.ascontiguousarray(event_layers, dtype=np.int32)
        rl = np.ascontiguousarray(retained_lengths, dtype=np.int64)
        return int(self.lib.orc_decode_seqused(original_length, decode_appended, el.size, _ptr(el, ctypes.c_int32),
                                               _ptr(rl, ctypes.c_int64), layer))

    def restrict_selection(self, sel: OracleSelection, veto, block_scores, block_size) -> OracleSelection:
        keep = sel.keep_mask.astype(np.uint8).copy()
        v = np.ascontiguousarray(veto, dtype=np.uint8)
        b = np.ascontiguousarray(block_scores, dtype=np.float32)
        info = _SelInfo(sel.cutoff_rank, sel.retained_count, sel.retention_ratio, sel.covered_mass,
                        int(sel.degenerate_keep_all))
        st = self.lib.orc_restrict_selection(_ptr(keep, ctypes.c_uint8), _ptr(v, ctypes.c_uint8),
                                             keep.size, _ptr(b, ctypes.c_float), b.size, block_size,
                                             ctypes.byref(info))
        _raise(st, "restrict_selection")
        return OracleSelection(keep, info.cutoff_rank, info.retained_count, info.retention_ratio,
                               info.covered_mass, bool(info.degenerate_keep_all))

    def compact(self, keep, cu_seqlens, planes, selected=None):
        """planes: list of 2-D arrays with T rows.  Returns (outs, cu_out, retained_index)."""
        keep = np.ascontiguousarray(keep, dtype=np.uint8)
        cu = np.ascontiguousarray(cu_seqlens, dtype=np.int64)
        R = cu.size - 1
        srcs = [np.ascontiguousarray(p) for p in planes]
        T = int(cu[-1])
        dsts = [np.zeros_like(s) for s in srcs]
        rb = np.array([s.strides[0] if s.ndim > 1 else s.itemsize for s in srcs], np.int64)
        sp = (ctypes.c_void_p * max(len(srcs), 1))(*[s.ctypes.data for s in srcs])
        dp = (ctypes.c_void_p * max(len(dsts), 1))(*[d.ctypes.data for d in dsts])
        sel = None if selected is None else np.ascontiguousarray(selected, dtype=np.uint8)
        cu_out = np.zeros(R + 1, np.int64)
        ridx = np.zeros(max(T, 1), np.int64)
        nout = ctypes.c_int64(0)
        st = self.lib.orc_compact(_ptr(keep, ctypes.c_uint8), _ptr(cu, ctypes.c_int64), R,
                                  _ptr(sel, ctypes.c_uint8) if sel is not None else None, len(srcs),
                                  sp, dp, _ptr(rb, ctypes.c_int64), _ptr(cu_out, ctypes.c_int64),
                                  _ptr(ridx, ctypes.c_int64), ctypes.byref(nout))
        _raise(st, "compact")
        n = int(nout.value)
        return [d[:n] for d in dsts], cu_out, ridx[:n]

    def rng_normal_array(self, seed: int, stream: int, count: int, stddev: float, first: int = 0) -> np.ndarray:
        """CounterRng(seed, stream).normal(first + j, stddev) for j < count (rng.cpp:34-40)."""
        out = np.empty(max(count, 1), np.float32)
        fn = self.lib.orc_rng_normal_fill
        fn.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64, ctypes.c_double,
                       ctypes.POINTER(ctypes.c_float)]
        fn.restype = None
        fn(self.lib.orc_rng_key(seed, stream), first, count, stddev, _ptr(out, ctypes.c_float))
        return out[:count]

    def c3_vectors(self, num_trials: int = 100000):
        """Acceptance criterion 3's inputs (acceptance_main.cpp:175-199), trials 0..num_trials-1:
        (scores concatenated fp32, offsets int64[num_trials+1], top_p fp32[num_trials])."""
        fn = self.lib.orc_c3_vector
        fn.argtypes = [ctypes.POINTER(ctypes.c_uint64), ctypes.c_int, ctypes.POINTER(ctypes.c_float),
                       ctypes.POINTER(ctypes.c_float)]
        fn.restype = ctypes.c_int64
        ctr = ctypes.c_uint64(0)
        buf = np.empty(4096, np.float32)
        p = ctypes.c_float(0)
        chunks, offsets, ps = [], [0], np.empty(num_trials, np.float32)
        for t in range(num_trials):
            n = fn(ctypes.byref(ctr), t, _ptr(buf, ctypes.c_float), ctypes.byref(p))
            chunks.append(buf[:n].copy())
            offsets.append(offsets[-1] + n)
            ps[t] = p.value
        return np.concatenate(chunks), np.asarray(offsets, np.int64), ps

    def c3_reference_blocks(self, scores, top_p: float) -> np.ndarray:
        """reference_blocks (acceptance_main.cpp:148-173) + the forced last token, as a mask."""
        s = np.ascontiguousarray(scores, dtype=np.float32)
        keep = np.zeros(max(s.size, 1), np.uint8)
        fn = self.lib.orc_c3_reference_blocks
        fn.argtypes = [ctypes.POINTER(ctypes.c_float), ctypes.c_int64, ctypes.c_double,
                       ctypes.POINTER(ctypes.c_uint8)]
        fn.restype = None
        fn(_ptr(s, ctypes.c_float), s.size, float(np.float32(top_p)), _ptr(keep, ctypes.c_uint8))
        return keep[:s.size]

    def rng_uniform(self, seed: int, stream: int, i: int) -> float:
        return float(self.lib.orc_rng_uniform(self.lib.orc_rng_key(seed, stream), i))

    def rng_bits(self, seed: int, stream: int, i: int) -> int:
        return int(self.lib.orc_rng_bits(self.lib.orc_rng_key(seed, stream), i))


class Ref(_Lib):
    def top_p_select_batch(self, scores, offsets, top_ps, **cfg):
        """The reference top_p_select on every vector scores[offsets[i]:offsets[i+1]] with
        top_p = top_ps[i]: (keep masks concatenated, cutoff ranks)."""
        s = np.ascontiguousarray(scores, dtype=np.float32)
        off = np.ascontiguousarray(offsets, dtype=np.int64)
        ps = np.ascontiguousarray(top_ps, dtype=np.float32)
        keep = np.zeros(max(s.size, 1), np.uint8)
        cut = np.zeros(max(ps.size, 1), np.int64)
        fn = self.lib.ref_top_p_select_batch
        P = ctypes.POINTER
        fn.argtypes = [P(ctypes.c_float), P(ctypes.c_int64), P(ctypes.c_float), ctypes.c_int32, P(_Cfg),
                       P(ctypes.c_uint8), P(ctypes.c_int64)]
        c = _cfg(**cfg)
        _raise(fn(_ptr(s, ctypes.c_float), _ptr(off, ctypes.c_int64), _ptr(ps, ctypes.c_float), ps.size,
                  ctypes.byref(c), _ptr(keep, ctypes.c_uint8), _ptr(cut, ctypes.c_int64)), "top_p_select_batch")
        return keep[:s.size], cut[:ps.size]

    """The unmodified reference core (oracle/_ref)."""

    def __init__(self, path: str = REF_SO):
        super().__init__(path, "ref")
        P = ctypes.POINTER
        self._fn("apply_drop", [P(ctypes.c_float), ctypes.c_int64, ctypes.c_int64, P(ctypes.c_uint8),
                                P(ctypes.c_float), P(ctypes.c_int64), P(ctypes.c_int64)])
        self._fn("reconstitute_sequence", [P(ctypes.c_float), ctypes.c_int64, ctypes.c_int64, ctypes.c_int32,
                                           P(P(ctypes.c_uint8)), P(P(ctypes.c_float)), P(ctypes.c_float),
                                           P(ctypes.c_int64)])
        self._fn("recompute_slots", [ctypes.c_int, ctypes.c_int, ctypes.c_int64, P(ctypes.c_int64), ctypes.c_int64,
                                     ctypes.c_int64, P(ctypes.c_int32), P(ctypes.c_int64)])
        self._fn("decode_seqused", [ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, P(ctypes.c_int32),
                                    P(ctypes.c_int64), ctypes.c_int32, P(ctypes.c_int64)])
        self._fn("patch_metadata", [P(ctypes.c_float), ctypes.c_int64, ctypes.c_int64, P(ctypes.c_int64),
                                    ctypes.c_int32, P(ctypes.c_uint8), P(ctypes.c_uint8),
                                    P(ctypes.c_uint8), P(ctypes.c_float), P(ctypes.c_int64)])
        self._fn("sharded_allreduce", [P(ctypes.c_float), ctypes.c_int64, P(ctypes.c_float),
                                       ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_int, P(_Cfg), ctypes.c_int, P(ctypes.c_float),
                                       P(ctypes.c_float)])
        self._fn("attention_readout", [P(ctypes.c_float), P(ctypes.c_int64), ctypes.c_int64, P(ctypes.c_float),
                                       P(ctypes.c_float), P(ctypes.c_int64), ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_int, ctypes.c_int64, P(ctypes.c_float)])
        self._fn("layer_flops", [ctypes.c_int32, ctypes.c_int64, P(_ModelCfg), P(ctypes.c_uint64)])
        self._fn("scoring_flops", [ctypes.c_int64, ctypes.c_int64, P(_ModelCfg), P(ctypes.c_uint64)])
        self._fn("validate_savings", [P(_ModelCfg), ctypes.c_int64, P(ctypes.c_int64), ctypes.c_int32,
                                      P(ctypes.c_int32), P(ctypes.c_int64), P(ctypes.c_int64), P(ctypes.c_double),
                                      ctypes.c_uint64, P(ctypes.c_uint64), P(ctypes.c_int32), P(ctypes.c_double)])
        self._fn("drop_layer_varlen", [P(ctypes.c_float), ctypes.c_int64, P(ctypes.c_float),
                                       ctypes.c_int64, P(ctypes.c_float), ctypes.c_int64,
                                       P(ctypes.c_int64), ctypes.c_int32, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_int, P(_Cfg), ctypes.c_int, P(ctypes.c_float),
                                       P(ctypes.c_uint8), P(ctypes.c_float), P(ctypes.c_int64)])

    def apply_drop(self, states: np.ndarray, keep):
        s = np.ascontiguousarray(states, dtype=np.float32)
        k = np.ascontiguousarray(keep, dtype=np.uint8)
        out = np.zeros_like(s)
        pos = np.zeros(s.shape[0], np.int64)
        n = ctypes.c_int64(0)
        st = self.lib.ref_apply_drop(_ptr(s, ctypes.c_float), s.shape[0], s.shape[1],
                                     _ptr(k, ctypes.c_uint8), _ptr(out, ctypes.c_float),
                                     _ptr(pos, ctypes.c_int64), ctypes.byref(n))
        _raise(st, "apply_drop")
        return out[: n.value], pos[: n.value]

    def reconstitute_sequence(self, prompt: np.ndarray, keeps, afters):
        """apply_drop per keep mask (replacing the active states by afters[d] after drop d),
        then reconstitute (propagation.cpp:79-100).  Returns (states, positions)."""
        pr = np.ascontiguousarray(prompt, dtype=np.float32)
        ks = [np.ascontiguousarray(k, dtype=np.uint8) for k in keeps]
        afs = [None if a is None else np.ascontiguousarray(a, dtype=np.float32) for a in afters]
        P = ctypes.POINTER
        kp = (P(ctypes.c_uint8) * len(ks))(*[_ptr(k, ctypes.c_uint8) for k in ks])
        ap = (P(ctypes.c_float) * len(ks))(*[_ptr(a, ctypes.c_float) if a is not None else None for a in afs])
        out = np.zeros_like(pr)
        pos = np.zeros(pr.shape[0], np.int64)
        st = self.lib.ref_reconstitute_sequence(_ptr(pr, ctypes.c_float), pr.shape[0], pr.shape[1], len(ks), kp, ap,
                                                _ptr(out, ctypes.c_float), _ptr(pos, ctypes.c_int64))
        _raise(st, "reconstitute_sequence")
        return out, pos

    def recompute_slots(self, num_layers: int, block_size: int, prealloc_len: int, retained, max_pages: int):
        """PagedKVCache::recompute_slots_after_drop for one request -> (tables [L, max_pages], slots [L, n])."""
        ret = np.ascontiguousarray(retained, dtype=np.int64)
        tables = np.zeros((num_layers, max_pages), np.int32)
        slots = np.zeros((num_layers, max(ret.size, 1)), np.int64)
        st = self.lib.ref_recompute_slots(num_layers, block_size, prealloc_len, _ptr(ret, ctypes.c_int64), ret.size,
                                          max_pages, _ptr(tables, ctypes.c_int32), _ptr(slots, ctypes.c_int64))
        _raise(st, "recompute_slots")
        return tables, slots[:, :ret.size]

    def decode_seqused(self, original_length: int, decode_appended: int, event_layers, retained_lengths, layer: int):
        el = np.ascontiguousarray(event_layers, dtype=np.int32)
        rl = np.ascontiguousarray(retained_lengths, dtype=np.int64)
        out = ctypes.c_int64(0)
        st = self.lib.ref_decode_seqused(original_length, decode_appended, el.size, _ptr(el, ctypes.c_int32),
                                         _ptr(rl, ctypes.c_int64), layer, ctypes.byref(out))
        _raise(st, "decode_seqused")
        return int(out.value)

    def attention_readout(self, q, q_pos, k, v, kv_pos, num_heads: int, num_kv_heads: int, window: int = 0):
        """attention_readout (model.cpp:215-263): q [rows, H*D], k/v [kv_rows, Hkv*D] fp32."""
        qa = np.ascontiguousarray(q, dtype=np.float32)
        ka = np.ascontiguousarray(k, dtype=np.float32)
        va = np.ascontiguousarray(v, dtype=np.float32)
        qp = np.ascontiguousarray(q_pos, dtype=np.int64)
        kp = np.ascontiguousarray(kv_pos, dtype=np.int64)
        D = qa.shape[1] // num_heads
        out = np.zeros_like(qa)
        st = self.lib.ref_attention_readout(_ptr(qa, ctypes.c_float), _ptr(qp, ctypes.c_int64), qa.shape[0],
                                            _ptr(ka, ctypes.c_float), _ptr(va, ctypes.c_float),
                                            _ptr(kp, ctypes.c_int64), ka.shape[0], num_heads, num_kv_heads, D,
                                            int(window), _ptr(out, ctypes.c_float))
        _raise(st, "attention_readout")
        return out

    def layer_flops(self, kind: int, tokens: int, cfg) -> int:
        c, _pat = _model_cfg(cfg)
        out = ctypes.c_uint64(0)
        _raise(self.lib.ref_layer_flops(int(kind), tokens, ctypes.byref(c), ctypes.byref(out)), "layer_flops")
        return int(out.value)

    def scoring_flops(self, effective_n: int, num_keys: int, cfg) -> int:
        c, _pat = _model_cfg(cfg)
        out = ctypes.c_uint64(0)
        _raise(self.lib.ref_scoring_flops(effective_n, num_keys, ctypes.byref(c), ctypes.byref(out)), "scoring_flops")
        return int(out.value)

    def validate_savings(self, cfg, original: int, accel_tokens, drops, scoring: int) -> dict:
        """validate_savings over a dense ledger at `original` tokens and an accelerated one
        (accel_tokens per layer; drops = [(layer, before, after, retention_ratio)])."""
        c, _pat = _model_cfg(cfg)
        at = np.ascontiguousarray(accel_tokens, dtype=np.int64)
        dl = np.ascontiguousarray([d[0] for d in drops] or [0], dtype=np.int32)
        db = np.ascontiguousarray([d[1] for d in drops] or [0], dtype=np.int64)
        da = np.ascontiguousarray([d[2] for d in drops] or [0], dtype=np.int64)
        dr = np.ascontiguousarray([d[3] for d in drops] or [0.0], dtype=np.float64)
        u = np.zeros(6, np.uint64)
        i = np.zeros(5, np.int32)
        f = np.zeros(2, np.float64)
        st = self.lib.ref_validate_savings(ctypes.byref(c), original, _ptr(at, ctypes.c_int64), len(drops),
                                           _ptr(dl, ctypes.c_int32), _ptr(db, ctypes.c_int64),
                                           _ptr(da, ctypes.c_int64), _ptr(dr, ctypes.c_double), scoring,
                                           _ptr(u, ctypes.c_uint64), _ptr(i, ctypes.c_int32), _ptr(f, ctypes.c_double))
        _raise(st, "validate_savings")
        return dict(dense_total=int(u[0]), accel_total=int(u[1]), scoring_overhead=int(u[2]),
                    measured_delta=int(u[3]), formula_delta=int(u[4]), closed_linear_form=int(u[5]),
                    exact_match=bool(i[0]), single_drop=bool(i[1]), drop_layer=int(i[2]),
                    layers_after_drop=int(i[3]), linear_form_exact=bool(i[4]),
                    retention_ratio=float(f[0]), attention_only_ratio=float(f[1]))

    def patch_metadata(self, tokens: np.ndarray, cu_seqlens, keep, selected, is_decode=None):
        t = np.ascontiguousarray(tokens, dtype=np.float32)
        cu = np.ascontiguousarray(cu_seqlens, dtype=np.int64)
        R = cu.size - 1
        k = np.ascontiguousarray(keep, dtype=np.uint8)
        sel = np.ascontiguousarray(selected, dtype=np.uint8)
        dec = None if is_decode is None else np.ascontiguousarray(is_decode, dtype=np.uint8)
        out = np.zeros_like(t)
        cu_out = np.zeros(R + 1, np.int64)
        st = self.lib.ref_patch_metadata(_ptr(t, ctypes.c_float), t.shape[0], t.shape[1],
                                         _ptr(cu, ctypes.c_int64), R, _ptr(k, ctypes.c_uint8),
                                         _ptr(sel, ctypes.c_uint8),
                                         _ptr(dec, ctypes.c_uint8) if dec is not None else None,
                                         _ptr(out, ctypes.c_float), _ptr(cu_out, ctypes.c_int64))
        _raise(st, "patch_metadata")
        return out[: cu_out[-1]], cu_out

    def sharded_allreduce(self, q, k, num_heads, num_kv_heads, tp_degree, **cfg):
        q = np.ascontiguousarray(q, dtype=np.float32)
        k = np.ascontiguousarray(k, dtype=np.float32)
        N = q.shape[0]
        D = q.shape[1] // num_heads
        c = _cfg(**cfg)
        nb = (N + c.block_size_g - 1) // c.block_size_g
        shards = np.zeros((tp_degree, nb), np.float32)
        red = np.zeros(nb, np.float32)
        st = self.lib.ref_sharded_allreduce(_ptr(q, ctypes.c_float), q.shape[1], _ptr(k, ctypes.c_float),
                                            k.shape[1], N, num_heads, num_kv_heads, D, ctypes.byref(c),
                                            tp_degree, _ptr(shards, ctypes.c_float),
                                            _ptr(red, ctypes.c_float))
        _raise(st, "sharded_allreduce")
        return shards, red

    def sharded_allreduce_mt(self, q_tail, k, num_heads, num_kv_heads, tp_degree, threads, **cfg):
        """sharded_block_scores + allreduce_scores with the shards on `threads` host threads
        (bitwise the sequential reference).  q_tail: the request's last >= n_eff query rows
        [rows, num_heads*D]; k: [N, num_kv_heads*D].  Returns (shards [tp, nb], reduced [nb])."""
        q = np.ascontiguousarray(q_tail, dtype=np.float32)
        k = np.ascontiguousarray(k, dtype=np.float32)
        N = k.shape[0]
        D = q.shape[1] // num_heads
        c = _cfg(**cfg)
        nb = (N + c.block_size_g - 1) // c.block_size_g
        shards = np.zeros((tp_degree, nb), np.float32)
        red = np.zeros(nb, np.float32)
        fn = self.lib.ref_sharded_allreduce_mt
        P = ctypes.POINTER
        fn.argtypes = [P(ctypes.c_float), ctypes.c_int64, ctypes.c_int64, P(ctypes.c_float), ctypes.c_int64,
                       ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int, P(_Cfg), ctypes.c_int, ctypes.c_int,
                       P(ctypes.c_float), P(ctypes.c_float)]
        _raise(fn(_ptr(q, ctypes.c_float), q.shape[1], q.shape[0], _ptr(k, ctypes.c_float), k.shape[1], N,
                  num_heads, num_kv_heads, D, ctypes.byref(c), tp_degree, threads,
                  _ptr(shards, ctypes.c_float), _ptr(red, ctypes.c_float)), "sharded_allreduce_mt")
        return shards, red

    def drop_unit(self, q_tail, k, hidden, num_heads, num_kv_heads, tp_degree=1, threads=1, **cfg):
        """One (request, drop layer) unit of the reference's varlen loop, hot path only
        (ref_drop_unit): returns (seconds, retained rows)."""
        q = np.ascontiguousarray(q_tail, dtype=np.float32)
        k = np.ascontiguousarray(k, dtype=np.float32)
        h = np.ascontiguousarray(hidden, dtype=np.float32)
        N = k.shape[0]
        D = q.shape[1] // num_heads
        c = _cfg(**cfg)
        fn = self.lib.ref_drop_unit
        P = ctypes.POINTER
        fn.argtypes = [P(ctypes.c_float), ctypes.c_int64, ctypes.c_int64, P(ctypes.c_float), ctypes.c_int64,
                       ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int, P(ctypes.c_float), ctypes.c_int64,
                       P(_Cfg), ctypes.c_int, ctypes.c_int, P(ctypes.c_int64), P(ctypes.c_double)]
        ret, sec = ctypes.c_int64(0), ctypes.c_double(0)
        _raise(fn(_ptr(q, ctypes.c_float), q.shape[1], q.shape[0], _ptr(k, ctypes.c_float), k.shape[1], N,
                  num_heads, num_kv_heads, D, _ptr(h, ctypes.c_float), h.shape[1], ctypes.byref(c), tp_degree,
                  threads, ctypes.byref(ret), ctypes.byref(sec)), "drop_unit")
        return float(sec.value), int(ret.value)

    def drop_layer_varlen(self, q, k, hidden, cu_seqlens, num_heads, num_kv_heads, threads=1, **cfg):
        """The reference's per-layer hot path over a varlen batch (score -> select -> compact)."""
        q = np.ascontiguousarray(q, dtype=np.float32)
        k = np.ascontiguousarray(k, dtype=np.float32)
        hid = np.ascontiguousarray(hidden, dtype=np.float32)
        cu = np.ascontiguousarray(cu_seqlens, dtype=np.int64)
        R = cu.size - 1
        T = int(cu[-1])
        D = q.shape[1] // num_heads
        c = _cfg(**cfg)
        G = c.block_size_g
        nbt = int(sum((int(cu[s + 1] - cu[s]) + G - 1) // G for s in range(R)))
        blk = np.zeros(max(nbt, 1), np.float32)
        keep = np.zeros(max(T, 1), np.uint8)
        hout = np.zeros_like(hid)
        cu_out = np.zeros(R + 1, np.int64)
        st = self.lib.ref_drop_layer_varlen(
            _ptr(q, ctypes.c_float), q.shape[1], _ptr(k, ctypes.c_float), k.shape[1],
            _ptr(hid, ctypes.c_float), hid.shape[1], _ptr(cu, ctypes.c_int64), R, num_heads,
            num_kv_heads, D, ctypes.byref(c), threads, _ptr(blk, ctypes.c_float),
            _ptr(keep, ctypes.c_uint8), _ptr(hout, ctypes.c_float), _ptr(cu_out, ctypes.c_int64))
        _raise(st, "drop_layer_varlen")
        return blk[:nbt], keep[:T], hout[: cu_out[-1]], cu_out


_port = None
_ref = None


def port() -> Port:
    global _port
    if _port is None:
        if not os.path.exists(PORT_SO):
            build()
        _port = Port()
    return _port


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref() -> Ref:
    global _ref
    if _ref is None:
        _ref = Ref()
    return _ref
