"""Markdown summary of one ncu `--set full --import-source on` report: key metrics, the
warp-stall breakdown and the hottest SASS lines per kernel (read here with ncu -i).

    python profiles/stall_summary.py REPORT.ncu-rep [kernel-regex] [top-N]
"""
from __future__ import annotations

import csv
import io
import subprocess
import sys

KEYS = [("gpu__time_duration.sum", "duration (us)"), ("sm__cycles_active.avg", "SM active cycles (avg)"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe % (active)"),
        ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
        ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
        ("dram__bytes_read.sum", "DRAM read (MB)"), ("dram__bytes_write.sum", "DRAM write (MB)"),
        ("launch__grid_size", "grid"), ("launch__block_size", "block"),
        ("launch__registers_per_thread", "registers/thread")]


def ncu_csv(args):
    out = subprocess.run(["ncu", "-i", *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep = sys.argv[1]
    kre = sys.argv[2] if len(sys.argv) > 2 else ".*"
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 12
    raw = ncu_csv([rep, "--page", "raw", "--kernel-name", f"regex:{kre}"])
    hdr = raw[0]
    seen = set()
    for r in raw[2:]:
        name = r[hdr.index("Kernel Name")]
        if name in seen:
            continue
        seen.add(name)
        print(f"### {name.split('(')[0]}\n")
        for k, label in KEYS:
            if k in hdr:
                print(f"- {label}: {r[hdr.index(k)]}")
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                try:
                    stalls.append((int(r[i]), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(v for v, _ in stalls) or 1
        print("- warp-state samples: " + ", ".join(f"{n} {100 * v / tot:.1f}%" for v, n in sorted(stalls, reverse=True)[:8]))
        src = ncu_csv([rep, "--page", "source", "--print-source", "sass", "--kernel-name", f"regex:{kre}"])
        blocks, cur = [], None
        for row in src:
            if row and row[0] == "Address":
                cur = [row]
                blocks.append(cur)
            elif cur is not None and len(row) > 3:
                cur.append(row)
        if blocks:
            h2, data = blocks[len(seen) - 1][0] if len(blocks) >= len(seen) else blocks[0][0], None
            b = blocks[len(seen) - 1] if len(blocks) >= len(seen) else blocks[0]
            h2, data = b[0], b[1:]
            isrc, iss = h2.index("Source"), h2.index("Warp Stall Sampling (All Samples)")
            stot = sum(int(x[iss] or 0) for x in data) or 1
            hot = sorted(range(len(data)), key=lambda i: -int(data[i][iss] or 0))[:top]
            print(f"- hottest SASS lines (share of {stot} samples):")
            for i in sorted(hot):
                print(f"  - [{i}] {100 * int(data[i][iss] or 0) / stot:.1f}% `{data[i][isrc].strip()[:70]}`")
        print()


if __name__ == "__main__":
    main()
