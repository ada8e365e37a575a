"""Dev probe: attention device time (CUDA graph of 10 calls) for small single-segment inputs."""
import sys
import torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import paper_2605_06221_b200 as up
from test_gpu_attention import _inputs

for L, Hq, Hkv in [(256, 32, 8), (512, 32, 8), (1472, 32, 8), (4096, 32, 8), (1472, 8, 2), (1472, 64, 8)]:
    q, k, v, pos, cu = _inputs([L], Hq, Hkv, 128, seed=3)
    q, k, v, pos, cu = q.cuda(), k.cuda(), v.cuda(), pos.cuda(), cu.cuda()
    out = up.attention_varlen(q, k, v, cu, pos)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        up.attention_varlen(q, k, v, cu, pos, out=out)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(10):
                up.attention_varlen(q, k, v, cu, pos, out=out)
        g.replay()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(s); g.replay(); e1.record(s)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 10 * 1e3
    fl = 4.0 * Hq * 128 * L * (L + 1) / 2
    print(f"L={L} Hq={Hq}: {us:.1f} us  {fl / us / 1e6:.1f} TFLOP/s", flush=True)
