"""Dev probe: the c2 drop-layer loop (LLaMA 4x32K, 32 layers) as M micro-batches of 4/M
requests, each on its own stream (its own CUDA graph), replayed concurrently.  Prints
ms per step and tokens/s for M = 1, 2, 4."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2605_06221_b200 as up  # noqa: E402
from paper_2605_06221_b200.synthetic import MODEL_SHAPES, make_batch  # noqa: E402

dev = torch.device("cuda", 0)
shp = MODEL_SHAPES["llama3.1-8b"]
Hq, Hkv, D, HID = shp["num_q_heads"], shp["num_kv_heads"], shp["head_dim"], shp["hidden"]
cfg = up.ScoreConfig(**bench.SPEC)
LAYERS, SETS = 32, int(os.environ.get("SETS", "8"))
lengths = [32768] * 4
for M in [int(x) for x in os.environ.get("MS", "1 2 4").split()]:
    groups = [lengths[i * len(lengths) // M:(i + 1) * len(lengths) // M] for i in range(M)]
    runners, graphs, streams = [], [], []
    for gi, gl in enumerate(groups):
        r = bench.LayerRunner(up, torch, "dp", shp, gl, cfg, dev, 1, 0)
        sets = [make_batch(gl, Hq, Hkv, D, HID, regime="planted", seed=100 * gi + s, device=dev) for s in range(SETS)]
        cu = sets[0].cu_seqlens
        s = torch.cuda.Stream(device=dev)

        def step(r=r, sets=sets, cu=cu):
            for l in range(LAYERS):
                r(sets[l % SETS], cu)
        with torch.cuda.stream(s):
            step()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            step()
        runners.append((r, sets))
        graphs.append(g)
        streams.append(s)
    main = torch.cuda.current_stream()
    for rep in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(main)
        for s, g in zip(streams, graphs):
            s.wait_event(e0)
            with torch.cuda.stream(s):
                g.replay()
        for s in streams:
            ev = torch.cuda.Event()
            ev.record(s)
            main.wait_event(ev)
        e1.record(main)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"M={M}: {ms:.3f} ms/step  {sum(lengths) * LAYERS / ms / 1e3:.1f} M tokens/s", flush=True)
    del runners, graphs, streams
    torch.cuda.empty_cache()
