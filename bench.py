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
                     public API, H2D/D2H inside the timed region), per-stage rooflines,
                     the CPU baseline (the reference on the host cores) and clocks.
  --impl reference   the unmodified reference C++ implementation (oracle/_ref, compiled
                     from /root/reference/proj/core/src) on the host cores, same metric.

Launched as `python bench.py --gpus N ...` or under torchrun for N > 1: each rank runs
its own batch (request sharding, weak scaling; no collective on the data path).
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

CONFIGS = {
    # name: (model, lengths, layers, cfg)
    "c1": ("llama3.1-8b", [4096], 1, dict(query_window_n=128, block_size_g=64, sink_count_a=128, top_p=0.99)),
    "c2": ("llama3.1-8b", [32768] * 4, 32, dict(query_window_n=128, block_size_g=64, sink_count_a=128, top_p=0.99)),
}
WORKLOAD_NAME = {
    "c1": "llama3.1-8b layer shape, 1x4096 tokens, 1 drop layer, score+select+compact",
    "c2": "llama3.1-8b layer shape, varlen 4x32768 tokens, 32 full-attn drop layers, score+select+compact",
}


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
    ap.add_argument("--profile-stages", action="store_true", default=True)
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


def ncu_traffic():
    """Per-launch DRAM bytes from the committed ncu --set full summary, if present."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return {}


# --------------------------------------------------------------------------- CPU reference
class CpuReferenceSample:
    """The reference (oracle/_ref) hot path on the host cores over a bounded sample of the
    same workload: `cores` concurrent 2048-token requests of the same model shape, each
    worker thread running score_tokens -> top_p_select on its request, then
    patch_metadata compacting the batch (scheduler.cpp:293-332)."""

    SEG = 2048

    def __init__(self, model, cfg, regime, seed=1234, threads=None):
        import numpy as np
        import oracle
        from paper_2605_06221_b200.synthetic import MODEL_SHAPES, make_batch

        self.shp = MODEL_SHAPES[model]
        self.cfg = cfg
        self.cores = threads or min(os.cpu_count() or 1, 64)
        if oracle.ref_available():
            self.impl, self.kind = oracle.ref(), "reference"
        else:
            self.impl, self.kind = oracle.port(), "port"
            self.cores = 1
        shp = self.shp
        sb = make_batch([self.SEG] * self.cores, shp["num_q_heads"], shp["num_kv_heads"], shp["head_dim"],
                        shp["hidden"], regime=regime, seed=seed, device="cpu")
        self.T = self.SEG * self.cores
        self.q = sb.q.float().reshape(self.T, -1).numpy()
        self.k = sb.k.float().reshape(self.T, -1).numpy()
        self.hid = sb.hidden.float().numpy()
        self.cu = sb.cu_seqlens.numpy().astype(np.int64)
        self.desc = (f"{self.cores} concurrent {self.SEG}-token requests ({model} shape, {regime}) through the "
                     f"reference score_tokens -> top_p_select -> patch_metadata, {self.cores} threads")

    def run(self):
        """Returns tokens/s of one pass over the sample."""
        shp = self.shp
        t0 = time.perf_counter()
        if self.kind == "reference":
            self.impl.drop_layer_varlen(self.q, self.k, self.hid, self.cu, shp["num_q_heads"],
                                        shp["num_kv_heads"], threads=self.cores, **self.cfg)
            T = self.T
        else:  # single-threaded restatement (no reference build available): one request
            seg = self.SEG
            tok, blk, _ = self.impl.score_tokens(self.q[:seg], self.k[:seg], shp["num_q_heads"],
                                                 shp["num_kv_heads"], **self.cfg)
            self.impl.top_p_select(blk, seg, **self.cfg)
            T = seg
        return T / (time.perf_counter() - t0)


def run_reference_arm(args):
    ws, rank, _ = dist_env()
    model, lengths, layers, cfg = CONFIGS[args.config]
    if rank != 0:
        return
    sample = CpuReferenceSample(model, cfg, args.regime)
    vals = []
    for i in range(args.warmup + args.steps):
        v = sample.run()
        if i >= args.warmup:
            vals.append(v)
    value = statistics.mean(vals)
    cores, kind, desc = sample.cores, sample.kind, sample.desc
    line = {
        "impl": "reference", "metric": "score+drop+compact tokens/s", "value": value, "unit": "tokens/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": None, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32 (fp64 accumulation)", "data": "synthetic",
        "config": {"workload": WORKLOAD_NAME[args.config], "regime": args.regime, **cfg},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": kind, "sample": desc},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- GPU arm
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2605_06221_b200 as up
    from paper_2605_06221_b200.synthetic import MODEL_SHAPES, make_batch

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)

    model, lengths, layers, cfgd = CONFIGS[args.config]
    shp = MODEL_SHAPES[model]
    Hq, Hkv, D, HID = shp["num_q_heads"], shp["num_kv_heads"], shp["head_dim"], shp["hidden"]
    cfg = up.ScoreConfig(**cfgd)
    R = len(lengths)
    T = sum(lengths)
    n = cfg.query_window_n

    # ---- activations: one set per layer (or --layer-sets distinct sets, cycled) ----
    free, _ = torch.cuda.mem_get_info(dev)
    per_set = T * (Hq * D + 2 * Hkv * D + HID) * 2 + T * 8
    n_sets = args.layer_sets or layers
    n_sets = max(1, min(n_sets, int((free * 0.8 - 3 * per_set) // per_set)))
    sets = []
    for s in range(n_sets):
        sb = make_batch(lengths, Hq, Hkv, D, HID, regime=args.regime, seed=1000 * rank + s, device=dev)
        sets.append(sb)
    cu = sets[0].cu_seqlens
    heads = up.HeadLayout(Hq, Hkv, D)
    plane_shapes = [(HID,), (Hkv, D), (Hkv, D), ()]
    plane_dtypes = [torch.bfloat16, torch.bfloat16, torch.bfloat16, torch.int64]
    layer = up.DropLayer(cfg, heads, T, R, plane_shapes, plane_dtypes, device=dev)

    def one_layer(sb):
        return layer(sb.q, sb.k, cu, [sb.hidden, sb.k, sb.v, sb.positions])

    def step():
        for l in range(layers):
            one_layer(sets[l % n_sets])

    # correctness guard on the first layer (device status), then warm-up
    one_layer(sets[0])
    layer.check()
    launches_per_layer = layer.last_launches
    use_graph = not args.no_graph
    graph = None
    stream = torch.cuda.Stream(device=dev)
    if use_graph:
        with torch.cuda.stream(stream):
            step()
        torch.cuda.synchronize(dev)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            step()
        run_step = graph.replay
    else:
        run_step = step

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            run_step()
    torch.cuda.synchronize(dev)
    layer.check()

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
    tokens_per_step = layers * T
    ms_per_step = ms / args.steps
    value = ws * tokens_per_step / (ms_per_step / 1e3)

    # retained fraction (planted regime) from the last layer
    rho = float(layer.out.num_out.item()) / T

    # ---- per-stage timing (events around each stage, same stream) ----
    stages = {}
    if args.profile_stages:
        names = ["score", "select", "compact"]
        evs = {nm: [] for nm in names}
        with torch.cuda.stream(stream):
            for l in range(layers):
                sb = sets[l % n_sets]
                e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
                e[0].record(stream)
                up.score_blocks_varlen(sb.q, sb.k, cu, cfg, heads, max_tokens=T, workspace=layer.ws,
                                       out=layer.scores)
                e[1].record(stream)
                up.select_varlen(layer.scores.block_scores, layer.scores.cu_blocks, cu, cfg, max_tokens=T,
                                 workspace=layer.ws, out=layer.sel)
                e[2].record(stream)
                up.compact_varlen(layer.sel.keep, cu, [sb.hidden, sb.k, sb.v, sb.positions], max_tokens=T,
                                  workspace=layer.ws, result=layer.out)
                e[3].record(stream)
                evs["score"].append((e[0], e[1]))
                evs["select"].append((e[1], e[2]))
                evs["compact"].append((e[2], e[3]))
        torch.cuda.synchronize(dev)
        for nm in names:
            stages[nm] = sum(a.elapsed_time(b) for a, b in evs[nm]) / layers
        retained = int(layer.out.num_out.item())
        hbm_peak, tf_peak, peak_kind = measured_peaks()
        flops = sum(2 * min(n, N) * N * D * Hq for N in lengths)
        row_bytes = HID * 2 + 2 * Hkv * D * 2 + 8
        comp_bytes = T * 1 + (R + 1) * 4 * 2 + retained * (2 * row_bytes + 4)
        traffic = ncu_traffic()
        score_ach = flops / (stages["score"] / 1e3) / 1e12
        comp_ach = comp_bytes / (stages["compact"] / 1e3) / 1e9
        stage_info = {
            "score": {"bound": "tensor", "achieved": score_ach, "peak": tf_peak, "unit": "TFLOP/s",
                      "frac": score_ach / tf_peak, "ms_per_layer": stages["score"],
                      "algorithmic_flops_per_layer": flops,
                      "traffic": traffic.get("score_tc_kernel")},
            "select": {"bound": "latency", "us_per_event": stages["select"] * 1e3, "requests": R},
            "compact": {"bound": "hbm", "achieved": comp_ach, "peak": hbm_peak, "unit": "GB/s",
                        "frac": comp_ach / hbm_peak, "ms_per_layer": stages["compact"],
                        "algorithmic_bytes_per_layer": comp_bytes,
                        "traffic": traffic.get("compact_scatter_kernel")},
        }
        dominant = "score" if stages["score"] >= stages["compact"] else "compact"
        d = stage_info[dominant]
        roofline = {"kernel": dominant, "bound": d["bound"], "achieved": d["achieved"], "peak": d["peak"],
                    "unit": d["unit"], "frac": d["frac"], "traffic": d["traffic"],
                    "peak_source": f"{peak_kind} (MEASURED_PEAKS.json burst)"}
    else:
        stage_info, roofline = {}, None

    # ---- e2e through the public API with host buffers ----
    e2e = None
    if args.e2e_steps > 0:
        src = sets[0]
        tails = []
        cu_h = cu.cpu().tolist()
        for r in range(R):
            s, e_ = cu_h[r], cu_h[r + 1]
            tails.append((max(s, e_ - n), e_))
        h_qt = [src.q[a:b].cpu().pin_memory() for a, b in tails]
        h_k = src.k.cpu().pin_memory()
        h_v = src.v.cpu().pin_memory()
        h_hid = src.hidden.cpu().pin_memory()
        h_pos = src.positions.cpu().pin_memory()
        h_cu = cu.cpu().pin_memory()
        d_q = torch.empty_like(src.q)
        d_k, d_v, d_hid, d_pos, d_cu = (torch.empty_like(src.k), torch.empty_like(src.v),
                                        torch.empty_like(src.hidden), torch.empty_like(src.positions),
                                        torch.empty_like(cu))
        o_keep = torch.empty(T, dtype=torch.uint8).pin_memory()
        o_cu = torch.empty(R + 1, dtype=torch.int32).pin_memory()
        o_cut = torch.empty(R, dtype=torch.int64).pin_memory()
        h2d = sum(t.numel() * t.element_size() for t in h_qt) + sum(
            t.numel() * t.element_size() for t in (h_k, h_v, h_hid, h_pos, h_cu))
        d2h = o_keep.numel() + o_cu.numel() * 4 + o_cut.numel() * 8

        def e2e_step():
            for l in range(layers):
                for (a, b), t in zip(tails, h_qt):
                    d_q[a:b].copy_(t, non_blocking=True)
                d_k.copy_(h_k, non_blocking=True)
                d_v.copy_(h_v, non_blocking=True)
                d_hid.copy_(h_hid, non_blocking=True)
                d_pos.copy_(h_pos, non_blocking=True)
                d_cu.copy_(h_cu, non_blocking=True)
                out = layer(d_q, d_k, d_cu, [d_hid, d_k, d_v, d_pos])
                o_keep.copy_(layer.sel.keep, non_blocking=True)
                o_cu.copy_(out.cu_seqlens, non_blocking=True)
                o_cut.copy_(layer.sel.cutoff_rank, non_blocking=True)

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
        if ws > 1:
            t = torch.tensor([ems], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": ws * tokens_per_step / (ems / args.e2e_steps / 1e3), "unit": "tokens/s",
               "h2d_bytes_per_step": h2d * layers, "d2h_bytes_per_step": d2h * layers,
               "steps": args.e2e_steps,
               "note": "per layer: H2D of q tail rows, K, V, hidden, positions, cu_seqlens from pinned "
                       "host memory; D2H of keep mask, new cu_seqlens, cutoff ranks"}

    # ---- CPU baseline (rank 0 only, N=1 semantics) ----
    cpu = None
    if rank == 0 and not args.skip_cpu:
        try:
            sample = CpuReferenceSample(model, cfgd, args.regime)
            v = sample.run()
            cpu = {"value": v, "unit": "tokens/s", "cores": sample.cores, "kind": sample.kind,
                   "sample": sample.desc}
        except Exception as exc:  # the baseline is reported, never fatal
            cpu = {"value": None, "unit": "tokens/s", "cores": None, "kind": None, "sample": f"failed: {exc}"}

    if rank == 0:
        line = {
            "metric": "score+drop+compact tokens/s", "value": value, "unit": "tokens/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic",
            "config": {"workload": WORKLOAD_NAME[args.config], "model_shape": model, "requests": R,
                       "tokens_per_request": lengths[0] if len(set(lengths)) == 1 else lengths,
                       "drop_layers": layers, "regime": args.regime, "retention_rho": rho,
                       "activation_sets": n_sets, "l2": "inputs larger than L2 (distinct per-layer sets)",
                       "cuda_graph": use_graph, "parallelism": f"request-sharded dp{ws}", **cfgd},
            "roofline": roofline, "stages": stage_info, "cpu_baseline": cpu, "e2e": e2e,
            "clocks": clk, "gpu_launches": launches_per_layer * layers * args.steps,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
