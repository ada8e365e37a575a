"""Dev probe: run up_attention_varlen on one shape, report time and max error vs torch."""
import sys, time
import torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import paper_2605_06221_b200 as up
from test_gpu_attention import _inputs, _torch_ref

LS = [int(x) for x in sys.argv[1].split(",")]
L, Hq, Hkv, D, W = max(LS), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
q, k, v, pos, cu = _inputs(LS, Hq, Hkv, D, seed=3)
q, k, v, pos, cu = q.cuda(), k.cuda(), v.cuda(), pos.cuda(), cu.cuda()
t = time.time()
out = up.attention_varlen(q, k, v, cu, pos, window=W)
torch.cuda.synchronize()
print("first call", time.time() - t, flush=True)
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(5):
    up.attention_varlen(q, k, v, cu, pos, window=W, out=out)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
fl = sum(4.0 * Hq * D * n * n / 2 for n in LS)
print(f"L={L} Hq={Hq} D={D}: {ms:.3f} ms  {fl / ms / 1e9:.1f} TFLOP/s", flush=True)
ref = _torch_ref(q, k, v, pos, cu.cpu(), W)
err = (out.float() - ref).abs()
print("max err", float(err.max()), "rel-bad", int((err > 2e-2 * (1 + ref.abs())).sum()), flush=True)
