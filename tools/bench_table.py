"""Dev: one line per bench log (value, score / select / compact / reconstitute stages, e2e,
clocks) for the DESIGN.md measurement table.  Usage: python tools/bench_table.py DIR"""
import json
import os
import sys

d = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
for name in ["bench_c1", "bench_c2", "bench_c2_stack2", "bench_c2_iid", "bench_c3", "bench_c3-rank", "bench_c4",
             "bench_c5", "bench_c5-mixed"]:
    f = os.path.join(d, name + ".log")
    if not os.path.exists(f):
        continue
    lines = [x for x in open(f).read().strip().splitlines() if x.startswith("{")]
    if not lines:
        print(f"{name:16s} (no JSON line)")
        continue
    j = json.loads(lines[-1])
    st = j.get("stages", {})
    sc, se, co, rc = (st.get(k, {}) for k in ("score", "select", "compact", "reconstitute"))
    e2e = (j.get("e2e") or {}).get("value")
    print(f"{name:16s} value {j['value'] / 1e6:7.1f}  score {sc.get('ms_per_layer', 0) * 1e3:7.1f} us "
          f"(tc {sc.get('frac', 0):.3f}, exp2 {sc.get('exp2', {}).get('frac', 0):.3f})  "
          f"select {se.get('us_per_event', 0):5.1f}  compact {co.get('ms_per_layer', 0) * 1e3:7.1f} us "
          f"({co.get('frac', 0):.3f})  recon {rc.get('ms_per_block', 0) * 1e3 if rc else 0:6.1f} us "
          f"({rc.get('frac', 0) if rc else 0:.3f})  e2e {(e2e or 0) / 1e6:5.2f}  "
          f"clk {j['clocks'].get('sm_mhz')} {j['clocks'].get('reasons')}")
