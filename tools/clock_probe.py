"""Dev: SM clock while the scorer stage runs back to back (nvidia-smi sampled at 50 ms)."""
import os, subprocess, sys, threading, time, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_06221_b200 as up
from paper_2605_06221_b200.synthetic import make_batch
sb = make_batch([32768] * 4, 32, 8, 128, 64, regime="planted", seed=1, device="cuda", with_v=False)
cfg = up.ScoreConfig(); h = up.HeadLayout(32, 8, 128)
out = up.score_blocks_varlen(sb.q, sb.k, sb.cu_seqlens, cfg, h)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(100): up.score_blocks_varlen(sb.q, sb.k, sb.cu_seqlens, cfg, h, out=out)
torch.cuda.synchronize()
p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active", "--format=csv,noheader,nounits", "-lms", "50"], stdout=subprocess.PIPE, text=True)
lines = []
th = threading.Thread(target=lambda: [lines.append(l.strip()) for l in p.stdout], daemon=True); th.start()
time.sleep(0.3)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(s):
    e0.record(s)
    for _ in range(200): g.replay()
    e1.record(s)
torch.cuda.synchronize()
p.terminate(); th.join(1)
print(f"{e0.elapsed_time(e1) / 20000:.4f} ms per scorer stage")
print("\n".join(lines[-40:]))
