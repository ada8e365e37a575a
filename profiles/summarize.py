"""Summarise the ncu outputs of profiles/run_profile.sh into committed files.

    python profiles/summarize.py gpurun_out r01 [SUFFIX CONFIG]   (e.g. _c3 c3: the Qwen3-Next capture)

writes profiles/launches_<tag>.csv (per-kernel share of the step from the launch list),
profiles/ncu_summary_<tag>.md (key metrics of the `--set full` captures) and
profiles/ncu_traffic.json (DRAM bytes per launch, read by bench.py for `roofline.traffic`).
"""
from __future__ import annotations

import collections
import csv
import io
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("sm__cycles_active.avg", "SM active cycles (avg)"),
    ("sm__cycles_active.max", "SM active cycles (max)"),
]


def short(name: str) -> str:
    base = name.split("(")[0]
    return base.replace("void ", "").replace("up::", "").strip()


def launch_shares(path: str):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        try:
            agg[short(r[ki])].append(float(r[vi].replace(",", "")))
        except ValueError:
            continue
    ours = {k: v for k, v in agg.items() if not k.startswith("at::") and "elementwise" not in k
            and "distribution" not in k and "at::native" not in k}
    tot = sum(sum(v) for v in ours.values())
    return sorted(((k, len(v), sum(v) / len(v), sum(v) / tot) for k, v in ours.items()), key=lambda x: -x[3])


def full_metrics(rep: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, data = rows[0], rows[1], rows[2:]
    res = []
    for r in data:
        d = {"kernel": short(r[h.index("Kernel Name")])}
        for m, _ in METRICS:
            if m in h:
                d[m] = (r[h.index(m)], units[h.index(m)])
        res.append(d)
    return res


def to_bytes(v, unit):
    x = float(v.replace(",", ""))
    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def main():
    src = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
    tag = sys.argv[2] if len(sys.argv) > 2 else "r01"
    suffix = sys.argv[3] if len(sys.argv) > 3 else ""
    config = sys.argv[4] if len(sys.argv) > 4 else "c2"
    workload = {"c2": "LLaMA-3.1-8B layer shape, 4x32K", "c3": "Qwen3-Next-80B-A3B full-attn layer, 1x128K, TP=8 sharded",
                "c4": "Gemma-3-12B layer shape, 16x64K"}.get(config, config)
    shares = launch_shares(os.path.join(src, f"launches{suffix}.csv"))
    with open(os.path.join(HERE, f"launches_{tag}{suffix}.csv"), "w") as f:
        f.write("kernel,launches,avg_ns,share_of_our_kernels\n")
        for k, n, avg, sh in shares:
            f.write(f"{k},{n},{avg:.0f},{sh:.4f}\n")
    full = full_metrics(os.path.join(src, f"prof_full{suffix}.ncu-rep"))
    attn = os.path.join(src, f"prof_attn{suffix}.ncu-rep")  # the drop-layer attention stage
    if os.path.exists(attn):
        full += full_metrics(attn)
    traffic = {}
    lines = [f"# ncu summary ({tag})", "",
             f"Command: `CONFIG={config} profiles/run_profile.sh` (bench.py --config {config}, {workload}, "
             "--no-graph, 2 activation sets); ncu --clock-control none.", "",
             "## Launch list (gpu__time_duration, cold-cache, serialised: compare shares)", "",
             "| kernel | launches | avg us | share of our kernels |", "|---|---|---|---|"]
    for k, n, avg, sh in shares:
        lines.append(f"| {k} | {n} | {avg / 1e3:.1f} | {sh:.3f} |")
    lines += ["", "## `--set full` captures", ""]
    for d in full:
        lines.append(f"### {d['kernel']}")
        for m, label in METRICS:
            if m in d:
                lines.append(f"- {label}: {d[m][0]} {d[m][1]}")
        if "dram__bytes_read.sum" in d:
            rd = to_bytes(*d["dram__bytes_read.sum"])
            wr = to_bytes(*d["dram__bytes_write.sum"])
            traffic.setdefault(d["kernel"], rd + wr)
        lines.append("")
    with open(os.path.join(HERE, f"ncu_summary_{tag}{suffix}.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    if config == "c2":  # bench.py's roofline.traffic is quoted for the default workload
        with open(os.path.join(HERE, "ncu_traffic.json"), "w") as f:
            json.dump(traffic, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
