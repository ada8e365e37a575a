#!/usr/bin/env python
"""UniPrefill score+drop+compact throughput on B200 (BASELINE.json `metric`).

Workload (BASELINE.json configs[1]): LLaMA-3.1-8B layer shape (32 q-heads, 8 kv-heads,
head_dim 128, hidden 4096), a continuous-batching varlen batch of 4 requests x 32K tokens,
all 32 layers as full-attention drop points, SPEC defaults n=128, G=64, A=128, p=0.99.
One step = the 32 drop layers, each scoring, selecting and compacting (hidden, K, V,
positions) the full batch entering it; tokens per step = 32 x 131072.  Inputs are
synthetic random-init bf16 activations (no network), a distinct activation set per layer
(each ~2.5 GB, far larger than the 126 MB L2).

Arms
  default            this repo's sm_100a kernels through the C ABI (CUDA-graph captured);
                     prints value (device-resident inputs), e2e (host buffers through the
                     public API, H2D/D2H inside the timed region), per-stage rooflines
                     (score, select, compact; plus the drop layer's attention over the
                     retained rows, reported beside the path and not part of `value`),
                     the CPU baseline (the reference on the host cores) and clocks.
  --impl reference   the unmodified reference C++ implementation (oracle/_ref, compiled
                     from /root/reference/proj/core/src) on the host cores, same metric.

Launched as `python bench.py --gpus N ...` or under torchrun for N > 1: each rank runs
its own batch (request sharding, weak scaling; no collective on the data path).  --config
c3 shards heads (TP): at N > 1 each rank scores its slice with the all-reduce fused into the
combine kernel over peer memory (UP_TP_REDUCE=nccl: NCCL all-gather + ordered reduce).
--config c1..c5 selects the other BASELINE.json configurations.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SPEC = dict(query_window_n=128, block_size_g=64, sink_count_a=128, top_p=0.99)
CONFIGS = {
    # name: (model shape, request lengths, drop layers per step, ScoreConfig, mode)
    #   mode "dp": request sharding (each rank its own batch: c1/c2 per rank, c5 LPT split)
    #   mode "tp": head sharding of one batch over the TP group (c3)
    "c1": ("llama3.1-8b", [4096], 1, SPEC, "dp"),
    "c2": ("llama3.1-8b", [32768] * 4, 32, SPEC, "dp"),
    # Qwen3-Next-80B-A3B: 48 layers, 3:1 linear/full -> 12 full-attention drop layers
    "c3": ("qwen3-next-80b-a3b", [131072], 12, SPEC, "tp"),
    # Gemma-3-12B: 48 layers, 5:1 sliding-window/full -> 8 full-attention drop layers, p=0.98
    "c4": ("gemma3-12b", [65536] * 16, 8, dict(SPEC, top_p=0.98), "dp"),
    # 64-request stream, N_r log-uniform in [4K, 128K] (seed 5), LPT-sharded over the ranks
    "c5": ("llama3.1-8b", "loguniform:64:4096:131072:5", 32, SPEC, "dp-split"),
    # one TP=8 rank's slice of c3 (2 q-heads, 1 kv-head, 128K) through the fused peer path
    "c3-rank": ("qwen3-next-80b-a3b", [131072], 12, SPEC, "tp-rank"),
    # envelope: c5's 64 prefills, each followed by 7 single-token decode segments (drop
    # disabled, passed through) -- 512 segments per launch
    "c5-mixed": ("llama3.1-8b", "mixed:64:4096:131072:5:7", 32, SPEC, "dp"),
}
# Block structure of each config (the reference's layer pattern, config.hpp:40 /
# model.hpp:48-50): a block is one full-attention drop layer followed by the sublayers that
# consume its compacted stream, and the block boundary reconstitutes the full stream
# (accelerated_prefill, propagation.cpp:258-283; Engine::run_batch, scheduler.cpp:283-361).
#   downstream: (kind, count) of the non-drop sublayers of a block -- their compute is the
#   model's, outside this path; "swa" layers own a paged KV cache, so the block recomputes
#   their Eq. 16 slot mapping from the compacted stream (up_slot_mapping);
#   reconstitute: scatter the block's retained rows back over the pre-drop hidden states at
#   the boundary (up_scatter_rows).  --stack S stacks S cascaded full-attention drop layers
#   per block (the reference's pure-full archetype, test_propagation.cpp:24-38): drop s+1
#   scores the stream drop s compacted, under drop s's device-resident cu_seqlens_out.
BLOCKS = {
    "c1": dict(downstream=("ffn", 0), reconstitute=False),   # one layer, no block boundary
    "c2": dict(downstream=("ffn", 0), reconstitute=True),    # LLaMA layer = [attention(drop), FFN]
    "c3": dict(downstream=("linear", 3), reconstitute=True),  # Qwen3-Next 3:1 = [full(drop), linear x3]
    "c3-rank": dict(downstream=("linear", 3), reconstitute=True),
    "c4": dict(downstream=("swa", 5), reconstitute=True),    # Gemma-3 5:1 = [full(drop), SWA x5]
    "c5": dict(downstream=("ffn", 0), reconstitute=True),
    "c5-mixed": dict(downstream=("ffn", 0), reconstitute=True),
}
KV_PAGE = 16  # paged-KV block size for the SWA layers' slot mapping (kvcache.hpp:36 default)
WORKLOAD_NAME = {
    "c1": "llama3.1-8b layer shape, 1x4096 tokens, 1 drop layer, score+select+compact",
    "c2": "llama3.1-8b layer shape, varlen 4x32768 tokens, 32 full-attn drop layers, score+select+compact",
    "c3": "qwen3-next-80b-a3b full-attn layer shape, 1x131072 tokens, 12 drop layers, TP=8 head-sharded "
          "scoring + ordered shard reduce, select, compact",
    "c4": "gemma3-12b layer shape, varlen 16x65536 tokens, 8 full-attn drop layers (p=0.98), "
          "score+select+compact",
    "c5": "llama3.1-8b layer shape, 64-request varlen stream (4K-128K log-uniform), 32 drop layers, "
          "LPT request-sharded, score+select+compact",
    "c3-rank": "qwen3-next-80b-a3b full-attn layer shape, ONE TP=8 rank's slice (2 q-heads, 1 kv-head) of "
               "1x131072 tokens, 12 drop layers: fused scorer+peer reduce (tp=1 group), select, compact",
    "c5-mixed": "llama3.1-8b layer shape, c5's 64 prefill requests each followed by 7 single-token decode "
                "segments (drop disabled): 512 segments, 32 drop layers, score+select+compact",
}


def config_lengths(spec):
    if isinstance(spec, str):
        kind, count, lo, hi, seed = spec.split(":")[:5]
        # the restatement below imports nothing of the product package (the reference arm
        # calls this too and must not map the repo's library)
        pre = loguniform_lengths_ref(int(count), int(lo), int(hi), int(seed))
        if kind == "mixed":  # each prefill followed by `dec` single-token decode segments
            dec = int(spec.split(":")[5])
            return [x for n in pre for x in [n] + [1] * dec]
        return pre
    return list(spec)


def config_drop_enabled(spec):
    """Per-segment drop_enabled flags (None = every segment is a prefill)."""
    if isinstance(spec, str) and spec.startswith("mixed:"):
        dec = int(spec.split(":")[5])
        return [x for _ in range(int(spec.split(":")[1])) for x in [1] + [0] * dec]
    return None


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=list(CONFIGS), default="c2")
    ap.add_argument("--regime", choices=["planted", "iid"], default="planted")
    ap.add_argument("--layer-sets", type=int, default=0, help="distinct activation sets (0 = one per layer)")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--no-stages", dest="profile_stages", action="store_false",
                    help="skip the per-stage timing (stages / roofline keys)")
    ap.add_argument("--query-window", type=int, default=0,
                    help="override the config's n (the paper's ablation: 32, 128, 512)")
    ap.add_argument("--block-size", type=int, default=0, help="override the config's G (ablation: 32, 64, 128)")
    ap.add_argument("--stack", type=int, default=1,
                    help="cascaded full-attention drop layers per block (drop s+1 scores drop s's compacted stream)")
    return ap.parse_args()


# --------------------------------------------------------------------------- dist helpers
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.th.join(timeout=2)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, val in zip(names, parts[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        loaded = [s for s in sm if smax and s > 0.5 * smax] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------------- peaks
def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), "measured"
    return 6650.0, 1590.0, "fallback"


def ncu_traffic(prefix):
    """Per-launch DRAM bytes (read + write) of the first kernel whose name starts with
    `prefix`, from the committed ncu --set full capture (profiles/ncu_traffic.json)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    for name, v in d.items():
        if name.startswith(prefix):
            return v
    return None


# --------------------------------------------------------------------------- CPU reference
# The reference arm imports nothing of this repo's product package (no repo .so is mapped):
# inputs come from numpy, the work from oracle/_ref (the unmodified reference build).
MODEL_SHAPES_REF = {  # the same layer shapes as paper_2605_06221_b200.synthetic.MODEL_SHAPES
    "llama3.1-8b": dict(num_q_heads=32, num_kv_heads=8, head_dim=128, hidden=4096),
    "qwen3-next-80b-a3b": dict(num_q_heads=16, num_kv_heads=2, head_dim=256, hidden=2048),
    "gemma3-12b": dict(num_q_heads=16, num_kv_heads=8, head_dim=256, hidden=3840),
}


def loguniform_lengths_ref(count, lo, hi, seed):
    """BASELINE config 5's request lengths (synthetic.loguniform_lengths restated)."""
    import torch
    g = torch.Generator().manual_seed(seed)
    u = torch.rand(count, generator=g, dtype=torch.float64)
    return [int(round(math.exp(math.log(lo) + float(x) * (math.log(hi) - math.log(lo))))) for x in u]


def cpu_model_name():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.lower().startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def _bf16_exact(x):
    """Round float32 to the nearest bf16 (ties to even), returned as float32."""
    import numpy as np
    u = x.astype(np.float32).view(np.uint32)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.view(np.float32)


class CpuReferenceUnits:
    """The reference hot path on the host cores, timed on units of the configured workload:
    a unit is one (request, drop layer) pair of the reference's varlen layer loop
    (scheduler.cpp:293-332) at the config's real request length -- score (the reference's
    TP=8 path sharded_block_scores + allreduce_scores, propagation.cpp:163-170, one shard per
    host thread) -> top_p_select -> apply_drop -> patch_metadata (oracle/_ref
    ref_drop_unit).  A step runs `units` units concurrently (units x 8 threads <= the host
    cores, bounded by memory); single_core() times one unit on ONE core through the
    unsharded score_tokens.  Inputs: numpy, bf16-exact, the planted/iid regimes of
    synthetic.make_batch restated (gamma 0.8, hot-block fraction 0.25)."""

    TP = 8

    def __init__(self, model, lengths, cfg, regime, seed=1234, rank_slice=False):
        import numpy as np
        import oracle
        if not oracle.ref_available():
            raise RuntimeError("oracle/_ref (the reference build) is missing")
        self.ref = oracle.ref()
        self.model, self.cfg, self.regime = model, cfg, regime
        self.shp = shp = dict(MODEL_SHAPES_REF[model])
        if rank_slice:
            # what ONE rank of the TP=8 group scores (c3-rank): its head slice, its two q-heads
            # as two shards on two threads (tp_sim.cpp:12-27 at T = 2 over the slice)
            hps = shp["num_q_heads"] // self.TP
            shp["num_kv_heads"] = max(1, shp["num_kv_heads"] * hps // shp["num_q_heads"])
            shp["num_q_heads"] = hps
            self.TP = hps
        self.nproc = os.cpu_count() or 1
        # distinct request lengths of the config, longest first (one input set per length)
        self.lengths = sorted(set(lengths), reverse=True)[:4]
        N = self.lengths[0]
        try:
            import psutil
            avail = psutil.virtual_memory().available
        except Exception:
            avail = 32 << 30
        unit_bytes = N * (4 * shp["hidden"] * 5 + 4 * shp["num_kv_heads"] * shp["head_dim"] * 3 +
                          4 * 128 * shp["num_q_heads"] // self.TP * 3)
        self.units = max(1, min(self.nproc // self.TP, int(avail * 0.5 // max(unit_bytes, 1)), 16))
        self.threads = self.units * self.TP
        rng = np.random.default_rng(seed)
        Hq, Hkv, D, HID = shp["num_q_heads"], shp["num_kv_heads"], shp["head_dim"], shp["hidden"]
        group = Hq // Hkv
        G = cfg["block_size_g"]
        n = cfg["query_window_n"]
        self.inputs = []
        for L in self.lengths:
            k = rng.standard_normal((L, Hkv, D), dtype=np.float32)
            qt = rng.standard_normal((min(n, L), Hq, D), dtype=np.float32)
            if regime == "planted":
                m = rng.standard_normal((Hkv, D), dtype=np.float32)
                qt += 0.8 * np.repeat(m, group, axis=0)[None]
                hot = np.repeat(rng.random((L + G - 1) // G) < 0.25, G)[:L]
                k[hot] += 0.8 * m[None]
            self.inputs.append((_bf16_exact(qt).reshape(len(qt), Hq * D), _bf16_exact(k).reshape(L, Hkv * D)))
        # hidden-state values do not change the reference's work: one shared bf16-exact buffer
        self.hidden = _bf16_exact(rng.standard_normal((N, HID), dtype=np.float32))
        self.desc = (f"(request, drop layer) units of the workload at their real lengths "
                     f"{self.lengths} ({model} shape{' -- one TP=8 rank slice' if rank_slice else ''}, "
                     f"{shp['num_q_heads']} q-heads / {shp['num_kv_heads']} kv-heads, {regime} bf16-exact inputs "
                     f"from numpy): the reference "
                     f"(oracle/_ref) score -> top_p_select -> apply_drop -> patch_metadata; {self.units} "
                     f"concurrent unit(s) per step, each scored through the reference's TP={self.TP} path "
                     f"(sharded_block_scores + allreduce_scores) with one shard per thread = {self.threads} "
                     f"threads on {self.nproc} host cores")
        self._next = 0

    def _unit(self, idx, tp, threads):
        qt, k = self.inputs[idx % len(self.inputs)]
        L = k.shape[0]
        shp = self.shp
        sec, kept = self.ref.drop_unit(qt, k, self.hidden[:L], shp["num_q_heads"], shp["num_kv_heads"], tp,
                                       threads, **self.cfg)
        return L, sec, kept

    def step(self):
        """One step: `units` concurrent units; returns (tokens/s, tokens, seconds)."""
        import concurrent.futures as cf
        idx = [self._next + u for u in range(self.units)]
        self._next += self.units
        t0 = time.perf_counter()
        with cf.ThreadPoolExecutor(self.units) as ex:
            res = list(ex.map(lambda i: self._unit(i, self.TP, self.TP), idx))
        sec = time.perf_counter() - t0
        tokens = sum(r[0] for r in res)
        return tokens / sec, tokens, sec

    def single_core(self):
        """One unit of the longest request on one core through the unsharded score_tokens."""
        L, sec, kept = self._unit(0, 1, 1)
        return L / sec, sec, L


def cpu_reference_report(units, step_values, single):
    value = statistics.mean(step_values)
    return {"value": value, "unit": "tokens/s", "cores": units.threads, "kind": "reference",
            "sample": units.desc, "nproc": units.nproc, "cpu_model": cpu_model_name(),
            "single_core": {"value": single[0], "unit": "tokens/s", "cores": 1, "seconds": single[1],
                            "tokens": single[2],
                            "path": "one unit of the longest request, unsharded score_tokens, one thread"}}


def run_reference_arm(args):
    ws, rank, _ = dist_env()
    if rank != 0:  # rank 0 alone measures the host; the other ranks exit without work
        return
    model, lspec, layers, cfg, _ = CONFIGS[args.config]
    if isinstance(lspec, str):
        _, count, lo, hi, seed = lspec.split(":")[:5]  # prefills (decode segments are not scored)
        lengths = loguniform_lengths_ref(int(count), int(lo), int(hi), int(seed))
    else:
        lengths = list(lspec)
    units = CpuReferenceUnits(model, lengths, cfg, args.regime, rank_slice=CONFIGS[args.config][4] == "tp-rank")
    vals = []
    for i in range(args.warmup + args.steps):
        v, _, _ = units.step()
        if i >= args.warmup:
            vals.append(v)
    single = units.single_core()
    cpu = cpu_reference_report(units, vals, single)
    value = cpu["value"]
    line = {
        "impl": "reference", "metric": "score+drop+compact tokens/s", "value": value, "unit": "tokens/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": None, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32 (fp64 accumulation)", "data": "synthetic",
        "config": workload_config(args.config, args.regime),
        "cpu_baseline": cpu,
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(name, regime):
    """The `config` object both arms print (identical, so the arms are comparable)."""
    model, lspec, layers, cfg, mode = CONFIGS[name]
    lengths = lspec if isinstance(lspec, str) else (lspec[0] if len(set(lspec)) == 1 else list(lspec))
    return {"workload": WORKLOAD_NAME[name], "model_shape": model,
            "requests": len(config_lengths(lspec)) if isinstance(lspec, str) else len(lspec),
            "tokens_per_request": lengths, "drop_layers": layers, "regime": regime,
            "unit": "(request, drop layer) pair; tokens = tokens entering the drop layer",
            "l2": "inputs larger than L2 (per-layer activation sets >> 126 MB)", **cfg}


# --------------------------------------------------------------------------- GPU arm
def attention_stage(up, runner, sb, cu, Hq, D, stream, dev, tf_peak, reps=5):
    """The drop layer's own attention over the retained rows (up_attention_varlen, SURVEY
    §8f row 1; propagation.cpp:195-205): run one drop layer on `sb`, gather the retained
    query rows (setup, untimed), then time the attention kernel over the compacted K, V and
    positions.  Reported beside the path, not part of `value`.  Algorithmic FLOPs: 4·D·Hq
    per (query row, visible key) -- QK^T and PV; causal, so row j of a segment of m
    retained rows sees j+1 keys."""
    torch = runner.torch
    with torch.cuda.stream(stream):
        runner(sb, cu)
        torch.cuda.synchronize(dev)
        L = runner.layer
        rows = int(L.out.num_out.item())
        idx = L.out.retained_index[:rows].long()
        q = torch.zeros(runner.T, Hq, D, dtype=torch.bfloat16, device=dev)
        q[:rows] = sb.q[idx]
        _, kc, vc, pc = L.out.planes
        heads = up.HeadLayout(Hq, runner.Hkv_local, D, gqa_group=runner.heads[0][2].gqa_group)
        out = torch.empty_like(q)
        cu_out = L.out.cu_seqlens
        lens = (cu_out[1:] - cu_out[:-1]).double()
        flops = float((4.0 * D * Hq * lens * (lens + 1) / 2).sum())

        def run():
            up.attention_varlen(q, kc, vc, cu_out, pc, heads=heads, max_tokens=runner.T, out=out)
        run()
        L.check()
        g = torch.cuda.CUDAGraph()  # device time only (a short launch is host-bound otherwise)
        with torch.cuda.graph(g, stream=stream):
            for _ in range(reps):
                run()
        g.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        g.replay()
        e1.record(stream)
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1) / reps
    ach = flops / (ms / 1e3) / 1e12
    return {"bound": "tensor", "achieved": ach, "peak": tf_peak, "unit": "TFLOP/s", "frac": ach / tf_peak,
            "ms_per_layer": ms, "algorithmic_flops_per_layer": flops, "rows": rows, "in_value": False,
            "note": "drop-layer attention over the retained rows (SURVEY 8f row 1), not part of value"}


class LayerRunner:
    """One drop layer (score -> [shard reduce] -> select -> compact) of the configured
    workload on this rank, through the public API (paper_2605_06221_b200.api)."""

    def __init__(self, up, torch, mode, shp, lengths, cfg, dev, world, rank, peer=None, drop_enabled=None):
        from paper_2605_06221_b200.distributed import head_slice
        # per-segment flags (decode segments pass through unscored, scheduler.cpp:59-62)
        self.en = None if drop_enabled is None else torch.tensor(drop_enabled, dtype=torch.uint8, device=dev)

        self.up, self.torch, self.mode, self.cfg, self.dev = up, torch, mode, cfg, dev
        Hq, Hkv, D, HID = shp["num_q_heads"], shp["num_kv_heads"], shp["head_dim"], shp["hidden"]
        self.T, self.R = sum(lengths), len(lengths)
        G = cfg.block_size_g
        self.nb = sum((n + G - 1) // G for n in lengths)
        self.world, self.rank = world, rank
        self.launches = 0
        if mode == "tp":
            # TP=8 head sharding (Eq. 15): at N=1 the eight shards are scored one after the
            # other on this GPU and summed by the ordered shard reduce; at N>1 every rank
            # scores its own head slice and the partials are all-reduced across ranks.
            self.tp = 8 if world == 1 else world
            slices = [head_slice(Hq, Hkv, t, self.tp) for t in range(self.tp)]
            self.shards = slices if world == 1 else [slices[rank]]
        elif mode == "tp-rank":
            # what ONE rank of the TP=8 group runs: its head slice only (rank 0's), scored
            # through the fused scorer + peer reduction on a one-rank group
            self.tp = 8
            self.shards = [head_slice(Hq, Hkv, 0, self.tp)]
        else:
            self.tp, self.shards = 1, [((0, Hq), (0, Hkv))]
        # planes compacted per layer: hidden, K, V of the local kv-heads, positions
        kb = min(sh[1][0] for sh in self.shards)
        ke = max(sh[1][1] for sh in self.shards)
        self.kv_range = (kb, ke)
        self.Hkv_local = ke - kb
        # At N>1 (tp) and in tp-rank mode the activation tensors hold only this rank's heads
        # (localize()).
        self.local = (mode == "tp" and world > 1) or mode == "tp-rank"
        self.heads = []
        for (qb, qe), (skb, ske) in self.shards:
            qi = (0, qe - qb) if self.local else (qb, qe)
            ki = (0, ske - skb) if self.local else (skb, ske)
            self.heads.append((qi, ki,
                               up.HeadLayout(qe - qb, ske - skb, D, gqa_group=Hq // Hkv, q_head_offset=qb,
                                             kv_head_offset=skb)))
        self.flops = sum(2 * min(cfg.query_window_n, N) * N * D * (qe - qb)
                         for N in lengths for (qb, qe), _ in self.shards)
        self.row_bytes = HID * 2 + 2 * self.Hkv_local * D * 2 + 8
        plane_shapes = [(HID,), (self.Hkv_local, D), (self.Hkv_local, D), ()]
        plane_dtypes = [torch.bfloat16, torch.bfloat16, torch.bfloat16, torch.int64]
        self.layer = up.DropLayer(cfg, up.HeadLayout(Hq, Hkv, D), self.T, self.R, plane_shapes, plane_dtypes,
                                  device=dev)
        self.peer = peer
        if peer is None and ((mode == "tp" and world > 1 and os.environ.get("UP_TP_REDUCE", "peer") == "peer")
                             or mode == "tp-rank"):
            from paper_2605_06221_b200.distributed import PeerScoreReducer
            self.peer = PeerScoreReducer(self.T // G + self.R + 1, device=dev)  # up_max_blocks
        if mode == "tp" and world == 1:
            nbmax = self.layer.scores.block_scores.numel()
            self.sharded = up.ShardedBlockScores(torch.empty(self.tp, nbmax, dtype=torch.float32, device=dev),
                                                 self.layer.scores.block_scores, self.layer.scores.cu_blocks)

    def localize(self, sb):
        """TP rank at N>1: keep only this rank's q-heads and kv-heads (what a rank holds)."""
        if self.local:
            (qb, qe), (kb, ke) = self.shards[0]
            sb.q = sb.q[:, qb:qe].contiguous()
            sb.k = sb.k[:, kb:ke].contiguous()
            sb.v = sb.v[:, kb:ke].contiguous()
        return sb

    def planes(self, sb, hidden=None, positions=None):
        """Planes compacted at the drop layer: the hidden states and positions of the stream
        entering it (default: the activation set's), the layer's K and V."""
        h = sb.hidden if hidden is None else hidden
        pos = sb.positions if positions is None else positions
        if self.local:
            return [h, sb.k, sb.v, pos]
        kb, ke = self.kv_range
        return [h, sb.k[:, kb:ke], sb.v[:, kb:ke], pos]

    def score(self, sb, cu):
        up, L = self.up, self.layer
        if self.mode not in ("tp", "tp-rank"):
            up.score_blocks_varlen(sb.q, sb.k, cu, self.cfg, L.heads, self.en, max_tokens=self.T, workspace=L.ws,
                                   out=L.scores)
            return up.lib.up_last_launch_count()
        if self.world == 1 and self.peer is None:
            # the whole TP group on one device: per-shard partials + ascending-shard sum in
            # one up_score_blocks_tp call (sharded_block_scores + allreduce_scores)
            up.score_blocks_tp(sb.q, sb.k, cu, self.cfg, self.tp, L.heads, max_tokens=self.T, workspace=L.ws,
                               out=self.sharded)
            return up.lib.up_last_launch_count()
        from paper_2605_06221_b200.distributed import allreduce_block_scores
        (qb, qe), (kb, ke), h = self.heads[0]
        if self.peer is not None:
            # this rank's heads scored with the all-reduce fused into the combine kernel
            # (partials stored straight into the peers' buffers, ascending-rank sum)
            self.peer.score_blocks(sb.q[:, qb:qe], sb.k[:, kb:ke], cu, self.cfg, h, max_tokens=self.T,
                                   workspace=L.ws, out=L.scores)
            return up.lib.up_last_launch_count()
        up.score_blocks_varlen(sb.q[:, qb:qe], sb.k[:, kb:ke], cu, self.cfg, h, max_tokens=self.T,
                               workspace=L.ws, out=L.scores)
        n = up.lib.up_last_launch_count()
        # UP_TP_REDUCE=nccl: NCCL all-gather + the ordered reduce kernel (bitwise allreduce_scores)
        allreduce_block_scores(L.scores.block_scores[:self.nb], deterministic=True)
        return n + up.lib.up_last_launch_count()

    def select(self, cu):
        L = self.layer
        self.up.select_varlen(L.scores.block_scores, L.scores.cu_blocks, cu, self.cfg, drop_enabled=self.en,
                              max_tokens=self.T, workspace=L.ws, out=L.sel)
        return self.up.lib.up_last_launch_count()

    def compact(self, sb, cu, hidden=None, positions=None):
        L = self.layer
        self.up.compact_varlen(L.sel.keep, cu, self.planes(sb, hidden, positions), drop_enabled=self.en,
                               max_tokens=self.T, workspace=L.ws, result=L.out, after_select=True)
        return self.up.lib.up_last_launch_count()

    def __call__(self, sb, cu, hidden=None, positions=None):
        self.launches = self.score(sb, cu) + self.select(cu) + self.compact(sb, cu, hidden, positions)


class BlockSchedule:
    """One step of the configured model on this rank: for every block, S cascaded drop
    layers (drop 0 on the full stream entering the block; drop s+1 on drop s's compacted
    planes under its device-resident cu_seqlens_out), the downstream sublayers' Eq. 16 slot
    mapping where they own a paged KV cache, and the reconstitution at the block boundary
    (the retained rows' states scattered back over the pre-drop hidden states, last drop
    first; propagation.cpp:79-100, scheduler.cpp:349-360).  Launch sizes depend only on
    capacities, so the whole step is one CUDA graph."""

    def __init__(self, up, torch, runners, resid, positions, cu, blocks, block_spec, sets, dev):
        self.up, self.torch = up, torch
        self.runners, self.resid, self.positions, self.cu = runners, resid, positions, cu
        self.blocks, self.S = blocks, len(runners)
        self.sets, self.n_sets = sets, len(sets)
        kind, count = block_spec["downstream"]
        self.reconstitute = block_spec["reconstitute"]
        self.slot_layers = count if kind == "swa" else 0
        self.launches = 0
        self.slots = self.tables = None
        if self.slot_layers:
            # identity page tables of the downstream SWA layers: request r's page i of layer
            # l is page (l * R + r) * max_pages + i
            R = cu.numel() - 1
            lens = (cu[1:] - cu[:-1]).tolist()
            max_pages = (max(lens) + KV_PAGE - 1) // KV_PAGE
            base = torch.arange(self.slot_layers * R, dtype=torch.int32, device=dev) * max_pages
            self.tables = (base[:, None] + torch.arange(max_pages, dtype=torch.int32, device=dev)[None]
                           ).reshape(self.slot_layers, R, max_pages).contiguous()
            self.slots = torch.empty(self.slot_layers, runners[0].T, dtype=torch.int64, device=dev)

    def layer_input(self, s):
        """(cu_seqlens, hidden, positions) of the stream entering drop s of a block."""
        if s == 0:
            return self.cu, self.resid, self.positions
        o = self.runners[s - 1].layer.out
        return o.cu_seqlens, o.planes[0], o.planes[3]

    def drop(self, b, s, stage=None):
        r = self.runners[s]
        act = self.sets[(b * self.S + s) % self.n_sets]
        cu, h, pos = self.layer_input(s)
        if stage is None:
            r(act, cu, h, pos)
            return r.launches
        if stage == "score":
            return r.score(act, cu)
        if stage == "select":
            return r.select(cu)
        return r.compact(act, cu, h, pos)

    def slot_map(self):
        if not self.slot_layers:
            return 0
        last = self.runners[-1].layer
        o = last.out
        self.up.slot_mapping(o.cu_seqlens, o.planes[3], self.tables, KV_PAGE, num_rows=o.num_out, out=self.slots,
                             workspace=last.ws)
        return self.up.lib.up_last_launch_count()

    def reconstitute_block(self):
        if not self.reconstitute:
            return 0
        n = 0
        for s in reversed(range(self.S)):
            o = self.runners[s].layer.out
            dst = self.resid if s == 0 else self.runners[s - 1].layer.out.planes[0]
            self.up.scatter_rows(o.retained_index, [o.planes[0]], [dst], num_rows=o.num_out)
            n += self.up.lib.up_last_launch_count()
        return n

    def step(self, record=None):
        n = 0
        for b in range(self.blocks):
            for s in range(self.S):
                n += self.drop(b, s)
                if record is not None:
                    record.append(self.runners[s].layer.out.num_out.clone())
            n += self.slot_map()
            n += self.reconstitute_block()
        self.launches = n

    def stage_pass(self, stage):
        for b in range(self.blocks):
            if stage in ("score", "select", "compact"):
                for s in range(self.S):
                    self.drop(b, s, stage)
            elif stage == "slots":
                self.slot_map()
            elif stage == "reconstitute":
                self.reconstitute_block()


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2605_06221_b200 as up
    from paper_2605_06221_b200.distributed import lpt_partition
    from paper_2605_06221_b200.synthetic import MODEL_SHAPES, make_batch

    ws, rank, local = dist_env()
    # one rank per GPU; UP_BENCH_BACKEND=gloo lets several ranks share one device (a
    # functional check of the multi-rank path on a single-GPU box, never a bench number)
    backend = os.environ.get("UP_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    model, lspec, layers, cfgd, mode = CONFIGS[args.config]
    if ws > 1:
        if mode == "tp-rank":
            raise SystemExit("--config c3-rank is the 1-GPU measurement of one TP rank's slice")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    elif mode == "tp-rank":
        # a one-rank group: the fused scorer + peer reduction runs exactly the kernels a TP
        # rank runs (its exchange is with itself)
        dist.init_process_group("gloo", store=dist.HashStore(), rank=0, world_size=1)

    shp = MODEL_SHAPES[model]
    Hq, Hkv, D, HID = shp["num_q_heads"], shp["num_kv_heads"], shp["head_dim"], shp["hidden"]
    cfg = up.ScoreConfig(**cfgd)
    all_lengths = config_lengths(lspec)
    if mode == "dp-split":   # a fixed request stream split across the ranks (LPT on N_r)
        lengths = [all_lengths[i] for i in lpt_partition(all_lengths, ws)[rank]]
        job_tokens, scaling = sum(all_lengths), "strong"
    elif mode == "tp":       # one batch, heads split across the ranks
        lengths = all_lengths
        job_tokens, scaling = sum(all_lengths), "strong"
        if ws > 1 and Hq % ws:
            raise SystemExit(f"--config {args.config}: {Hq} q-heads do not split over {ws} ranks")
    else:                    # every rank runs its own batch (tp-rank: one rank's slice)
        lengths = all_lengths
        job_tokens, scaling = ws * sum(all_lengths), "weak"
    R, T = len(lengths), sum(lengths)
    n = cfg.query_window_n
    S = max(1, args.stack)
    if layers % S:
        raise SystemExit(f"--stack {S} does not divide the config's {layers} drop layers")
    blocks = layers // S
    block_spec = BLOCKS[args.config]
    en = config_drop_enabled(lspec)
    runners = [LayerRunner(up, torch, mode, shp, lengths, cfg, dev, ws, rank, drop_enabled=en)]
    runners += [LayerRunner(up, torch, mode, shp, lengths, cfg, dev, ws, rank, peer=runners[0].peer,
                            drop_enabled=en) for _ in range(S - 1)]  # one exchange buffer per rank
    runner = runners[0]

    # ---- activations: one set per drop layer (or --layer-sets distinct sets, cycled) ----
    # Per-layer q, k, v (the layer's own projections); the hidden states are ONE residual
    # stream per rank that every block compacts and reconstitutes.
    free, _ = torch.cuda.mem_get_info(dev)
    per_set = T * (Hq * D + 2 * Hkv * D) * 2 + T * 8
    n_sets = args.layer_sets or layers
    n_sets = max(1, min(n_sets, int((free * 0.6 - 3 * per_set - T * HID * 2) // per_set)))
    sets = [runner.localize(make_batch(lengths, Hq, Hkv, D, HID, regime=args.regime,
                                       seed=1000 * (rank if mode not in ("tp", "tp-rank") else 0) + s, device=dev,
                                       with_hidden=False))
            for s in range(n_sets)]
    gen = torch.Generator(device=dev)
    gen.manual_seed(7 + rank)
    resid = torch.randn(T, HID, generator=gen, device=dev, dtype=torch.float32).to(torch.bfloat16)
    for sb in sets:
        sb.hidden = resid
    torch.cuda.empty_cache()
    cu = sets[0].cu_seqlens
    sched = BlockSchedule(up, torch, runners, resid, sets[0].positions, cu, blocks, block_spec, sets, dev)
    resid_ref = resid.clone()

    # correctness guard on the first block + the retained count of every drop layer of the
    # step (data-dependent with --stack: tokens entering drop s+1 = drop s's num_out)
    record = []
    sched.step(record)
    for r in runners:
        r.layer.check()
    retained = [int(x.item()) for x in record]
    if block_spec["reconstitute"] and not torch.equal(resid, resid_ref):
        # no model compute between the drop and the boundary: reconstitution must restore
        # the residual stream bit for bit (reconstitute, propagation.cpp:79-100)
        raise SystemExit("reconstitution did not restore the residual stream")
    del resid_ref
    entering = []
    for b in range(blocks):
        entering.append(T)
        entering.extend(retained[b * S:(b + 1) * S - 1])
    # tokens entering drop layers per step over the job: the ranks' own streams summed
    # (request sharding), or the one stream every TP rank scores a head slice of
    tokens_per_step = float(sum(entering))
    if ws > 1 and mode != "tp":
        t = torch.tensor([tokens_per_step], dtype=torch.float64, device=dev)
        dist.all_reduce(t)
        tokens_per_step = float(t.item())
    launches_per_step = sched.launches
    use_graph = not args.no_graph and not (mode == "tp" and ws > 1 and runner.peer is None)
    stream = torch.cuda.Stream(device=dev)
    if use_graph:
        with torch.cuda.stream(stream):
            sched.step()
        torch.cuda.synchronize(dev)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            sched.step()
        run_step = graph.replay
    else:
        run_step = sched.step

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            run_step()
    torch.cuda.synchronize(dev)
    for r in runners:
        r.layer.check()

    # ---- timed region (device-resident inputs) ----
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        ev0.record(stream)
        for _ in range(args.steps):
            run_step()
        ev1.record(stream)
    torch.cuda.synchronize(dev)
    ms = ev0.elapsed_time(ev1)
    clk = clocks.stop()
    if ws > 1:
        dist.barrier()
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    value = tokens_per_step / (ms_per_step / 1e3)
    rho = float(runner.layer.out.num_out.item()) / T

    # ---- per-stage timing: each stage over all layers captured in its own CUDA graph
    # (device time only, no host launch gaps), replayed between events on the stream ----
    stage_info, roofline = {}, None
    if args.profile_stages:
        names = ["score", "select", "compact"]
        if sched.slot_layers:
            names.append("slots")
        if block_spec["reconstitute"]:
            names.append("reconstitute")
        stages = {}
        # short configs (C1: one layer) repeat the pass inside the graph so a stage's time
        # is its kernels' device time, not one graph launch's latency
        reps = max(1, 32 // layers) if use_graph else 1
        for nm in names:
            def stage_pass(nm=nm):
                sched.stage_pass(nm)
            with torch.cuda.stream(stream):
                stage_pass()
            torch.cuda.synchronize(dev)
            if use_graph:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=stream):
                    for _ in range(reps):
                        stage_pass()
                run = g.replay
            else:
                run = stage_pass
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                run()
                e0.record(stream)
                run()
                e1.record(stream)
            torch.cuda.synchronize(dev)
            stages[nm] = e0.elapsed_time(e1) / reps / (layers if nm in ("score", "select", "compact") else blocks)
            del run
        hbm_peak, tf_peak, peak_kind = measured_peaks()

        def prof_traffic(prefix):  # the committed ncu capture is of the c2 workload
            return ncu_traffic(prefix) if args.config == "c2" and S == 1 else None

        # per drop layer averages over the step's drop layers
        mean_in = sum(entering) / len(entering)
        mean_kept = sum(retained) / len(retained)
        flops = runner.flops * mean_in / T  # scoring_flops is linear in N_r at N_r >= n
        comp_bytes = mean_in * 1 + (R + 1) * 4 * 2 + mean_kept * (2 * runner.row_bytes + 4)
        score_ach = flops / (stages["score"] / 1e3) / 1e12
        comp_ach = comp_bytes / (stages["compact"] / 1e3) / 1e9
        # The scorer's second bound: one exp2 per (row, key, head) logit -- flops / (2 D) --
        # against MUFU.EX2 at 16 / clk / SM (the epilogue moves part of them to the FMA
        # pipe at D = 128, so frac may approach or pass 1 without being wrong).
        f_mhz = clk.get("sm_mhz") or clk.get("sm_max_mhz") or 1965.0
        exps = flops / (2 * D)
        exp_ach = exps / (stages["score"] / 1e3) / 1e9
        exp_peak = torch.cuda.get_device_properties(dev).multi_processor_count * 16 * f_mhz * 1e6 / 1e9
        # and its third: every shard scored reads its kv-heads' K once (HBM)
        k_bytes = mean_in * sum(ske - skb for _, (skb, ske) in runner.shards) * D * 2
        k_ach = k_bytes / (stages["score"] / 1e3) / 1e9
        stage_info = {
            "score": {"bound": "tensor", "achieved": score_ach, "peak": tf_peak, "unit": "TFLOP/s",
                      "frac": score_ach / tf_peak, "ms_per_layer": stages["score"],
                      "algorithmic_flops_per_layer": flops,
                      "traffic": prof_traffic("score_tcw"),
                      "exp2": {"bound": "mufu", "achieved": exp_ach, "peak": exp_peak, "unit": "Gexp2/s",
                               "frac": exp_ach / exp_peak, "exp2_per_layer": exps,
                               "peak_basis": f"SMs x 16 MUFU.EX2/clk x {f_mhz:.0f} MHz (sampled SM clock)"},
                      "k_stream": {"bound": "hbm", "achieved": k_ach, "peak": hbm_peak, "unit": "GB/s",
                                   "frac": k_ach / hbm_peak, "k_bytes_per_layer": k_bytes}},
            "select": {"bound": "latency", "us_per_event": stages["select"] * 1e3, "requests": R},
            "compact": {"bound": "hbm", "achieved": comp_ach, "peak": hbm_peak, "unit": "GB/s",
                        "frac": comp_ach / hbm_peak, "ms_per_layer": stages["compact"],
                        "algorithmic_bytes_per_layer": comp_bytes,
                        "traffic": prof_traffic("compact_copy")},
        }
        if "reconstitute" in stages:
            # per block: every drop's retained hidden rows read + written, and its index
            rec_bytes = sum(retained[:S]) * (2 * HID * 2 + 4)
            ach = rec_bytes / (stages["reconstitute"] / 1e3) / 1e9
            stage_info["reconstitute"] = {"bound": "hbm", "achieved": ach, "peak": hbm_peak, "unit": "GB/s",
                                          "frac": ach / hbm_peak, "ms_per_block": stages["reconstitute"],
                                          "algorithmic_bytes_per_block": rec_bytes}
        if "slots" in stages:
            stage_info["slots"] = {"bound": "latency", "us_per_block": stages["slots"] * 1e3,
                                   "downstream_layers": sched.slot_layers}
        dominant = "score" if stages["score"] >= stages["compact"] else "compact"
        d = stage_info[dominant]
        roofline = {"kernel": dominant, "bound": d["bound"], "achieved": d["achieved"], "peak": d["peak"],
                    "unit": d["unit"], "frac": d["frac"], "traffic": d["traffic"],
                    "peak_source": f"{peak_kind} (MEASURED_PEAKS.json burst)"}
        if dominant == "score":  # the scorer's other bounds (stages.score has the details)
            roofline["also"] = {"mufu_exp2_frac": d["exp2"]["frac"], "k_stream_hbm_frac": d["k_stream"]["frac"]}
        if not runner.local and S == 1:
            stage_info["attention"] = attention_stage(up, runner, sets[0], cu, Hq, D, stream, dev, tf_peak)
            stage_info["attention"]["traffic"] = prof_traffic("attention")

    # ---- e2e through the public API with host buffers ----
    # Inputs start in pinned host memory every step.  The scorer needs the query-window rows
    # and all of K on the device (TMA), so those are copied H2D; the residual stream, V and
    # positions stay in pinned host memory: the compaction kernel reads the retained rows in
    # place over PCIe and the reconstitution scatter writes them back in place, so only
    # retained rows cross the bus (counted in h2d/d2h_bytes_per_step).
    e2e = None
    if args.e2e_steps > 0 and S == 1:
        src = sets[0]
        cu_h = cu.cpu().tolist()
        tails = [(max(cu_h[r], cu_h[r + 1] - n), cu_h[r + 1]) for r in range(R)]
        h_qt = [src.q[a:b].cpu().pin_memory() for a, b in tails]
        h_k, h_v, h_hid, h_pos, h_cu = (x.cpu().pin_memory() for x in
                                        (src.k, src.v, resid, src.positions, cu))
        d_in = type(src)(torch.empty_like(src.q), torch.empty_like(src.k), h_v, h_hid, h_pos,
                         torch.empty_like(cu), src.lengths)
        o_keep = torch.empty(T, dtype=torch.uint8).pin_memory()
        o_cu = torch.empty(R + 1, dtype=torch.int32).pin_memory()
        o_cut = torch.empty(R, dtype=torch.int64).pin_memory()
        h2d_copies = sum(t.numel() * t.element_size() for t in h_qt) + sum(
            t.numel() * t.element_size() for t in (h_k, h_cu))
        host_row_bytes = HID * 2 + runner.Hkv_local * D * 2 + 8  # hidden + V + position per retained row
        d2h = o_keep.numel() + o_cu.numel() * 4 + o_cut.numel() * 8
        L0 = runner.layer
        # Double-buffered inputs: the next layer's query-window rows, K and cu_seqlens are
        # copied H2D on a side stream while this layer scores, compacts and scatters (the
        # scatter's zero-copy writes travel D2H, so the copy engines and the PCIe link run
        # both directions at once); a buffer is refilled only after the layer using it has
        # compacted (its K plane is a compaction source).
        bufs = [d_in, type(src)(torch.empty_like(src.q), torch.empty_like(src.k), h_v, h_hid, h_pos,
                                torch.empty_like(cu), src.lengths)]
        cs = torch.cuda.Stream(device=dev)
        ev_copied = [torch.cuda.Event(), torch.cuda.Event()]
        ev_free = [torch.cuda.Event(), torch.cuda.Event()]
        for ev in ev_free:
            ev.record(stream)

        def copy_in(i):
            buf = bufs[i]
            with torch.cuda.stream(cs):
                cs.wait_event(ev_free[i])
                for (a, b), t in zip(tails, h_qt):
                    buf.q[a:b].copy_(t, non_blocking=True)
                buf.k.copy_(h_k, non_blocking=True)
                buf.cu_seqlens.copy_(h_cu, non_blocking=True)
                ev_copied[i].record(cs)

        def e2e_step():
            start = torch.cuda.Event()
            start.record(stream)
            cs.wait_event(start)  # this step's copies start after the step does
            copy_in(0)
            for l in range(layers):
                i = l % 2
                if l + 1 < layers:
                    copy_in((l + 1) % 2)
                stream.wait_event(ev_copied[i])
                buf = bufs[i]
                runner(buf, buf.cu_seqlens)
                ev_free[i].record(stream)
                if block_spec["reconstitute"]:
                    up.scatter_rows(L0.out.retained_index, [L0.out.planes[0]], [h_hid], num_rows=L0.out.num_out)
                o_keep.copy_(L0.sel.keep, non_blocking=True)
                o_cu.copy_(L0.out.cu_seqlens, non_blocking=True)
                o_cut.copy_(L0.sel.cutoff_rank, non_blocking=True)

        with torch.cuda.stream(stream):
            e2e_step()
            torch.cuda.synchronize(dev)
            if ws > 1:
                dist.barrier()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(args.e2e_steps):
                e2e_step()
            b.record(stream)
        torch.cuda.synchronize(dev)
        ems = a.elapsed_time(b)
        retained_e2e = int(L0.out.num_out.item())
        # correctness of the zero-copy path: same compacted hidden rows as the device path,
        # and the host residual stream restored by the in-place reconstitution
        ref_rows = resid[L0.out.retained_index[:retained_e2e].long()]
        if not torch.equal(L0.out.planes[0][:retained_e2e], ref_rows):
            raise SystemExit("e2e: zero-copy compaction differs from the device-resident path")
        if block_spec["reconstitute"] and not torch.equal(h_hid, resid.cpu()):
            raise SystemExit("e2e: host reconstitution did not restore the residual stream")
        if ws > 1:
            t = torch.tensor([ems], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        h2d = h2d_copies + retained_e2e * host_row_bytes
        d2h_all = d2h + (retained_e2e * HID * 2 if block_spec["reconstitute"] else 0)
        e2e = {"value": job_tokens * layers / (ems / args.e2e_steps / 1e3), "unit": "tokens/s",
               "h2d_bytes_per_step": h2d * layers, "d2h_bytes_per_step": d2h_all * layers,
               "steps": args.e2e_steps,
               "pcie_gbs": (h2d + d2h_all) * layers / (ems / args.e2e_steps / 1e3) / 1e9,
               "note": "per layer: H2D copies of the query-window rows, K and cu_seqlens from pinned host "
                       "memory (double-buffered on a side stream: the next layer's copy overlaps this layer); "
                       "residual stream, V and positions read in place from pinned host memory by the "
                       "compaction kernel (retained rows only); reconstitution scatters the retained hidden "
                       "rows back into the pinned host residual stream; D2H of keep mask, new cu_seqlens, "
                       "cutoff ranks"}

    # ---- CPU baseline (rank 0 only, N=1 semantics) ----
    cpu = None
    if rank == 0 and ws == 1 and not args.skip_cpu:  # reported at N=1 only
        try:  # one step of the reference arm's units (all cores) + one unit on one core
            units = CpuReferenceUnits(model, all_lengths, cfgd, args.regime, rank_slice=mode == "tp-rank")
            cpu = cpu_reference_report(units, [units.step()[0]], units.single_core())
            del units
        except Exception as exc:  # the baseline is reported, never fatal
            cpu = {"value": None, "unit": "tokens/s", "cores": None, "kind": None, "sample": f"failed: {exc}"}

    if rank == 0:
        if mode == "tp":
            par = f"tp{runner.tp} head-sharded" + (" (whole TP group on 1 GPU: per-shard partials + ordered "
                                                   "shard sum in one up_score_blocks_tp call)" if ws == 1 else
                                                   (" (fused scorer + peer-memory reduce)" if runner.peer else
                                                    " (NCCL all-gather + ordered reduce)"))
        elif mode == "tp-rank":
            par = "one rank of tp8 (rank 0's heads; fused scorer + peer-memory reduce on a one-rank group)"
        elif mode == "dp-split":
            par = f"LPT request-sharded over {ws} GPU(s)"
        else:
            par = f"request-sharded dp{ws}"
        kind, count = block_spec["downstream"]
        line = {
            "metric": "score+drop+compact tokens/s", "value": value, "unit": "tokens/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic",
            "config": workload_config(args.config, args.regime),
            "details": {"requests_per_rank": R, "tokens_per_rank": T, "retention_rho": rho,
                        "activation_sets": n_sets,
                        "blocks": blocks, "drops_per_block": S,
                        "block": f"{S} x full-attn drop layer" + (f" + {count} x {kind} sublayers" if count else "")
                                 + (" + reconstitution at the boundary" if block_spec["reconstitute"] else ""),
                        "tokens_entering_drops_per_step": sum(entering),
                        "retained_per_drop_first_block": retained[:S],
                        "seeds": "make_batch seed = 1000 * rank + activation-set index; residual stream seed 7 + rank "
                                 "(torch.Generator on the device)",
                        "l2": "inputs larger than L2 (distinct per-layer activation sets, each >> 126 MB)",
                        "cuda_graph": use_graph, "parallelism": par},
            "roofline": roofline, "stages": stage_info, "cpu_baseline": cpu, "e2e": e2e,
            "clocks": clk, "gpu_launches": launches_per_step * args.steps,
        }
        print(json.dumps(line), flush=True)
    if runner.peer is not None:
        for r in runners:
            r.layer.check()
        runner.peer.check()
        runner.peer.close()
    if dist.is_initialized():
        dist.destroy_process_group()


def main():
    args = parse()
    if args.query_window or args.block_size:  # ablation shapes: both arms see the same config
        model, lspec, layers, cfgd, mode = CONFIGS[args.config]
        cfgd = dict(cfgd)
        if args.query_window:
            cfgd["query_window_n"] = args.query_window
        if args.block_size:
            cfgd["block_size_g"] = args.block_size
        CONFIGS[args.config] = (model, lspec, layers, cfgd, mode)
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
