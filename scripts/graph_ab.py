"""A/B: the garden step (S1–S9) launched eagerly vs replayed from one CUDA graph.
Prints one JSON line with the median per-step ms of each (CUDA events, 20 steps, 3 rounds)."""
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2506_12727_b200 import mvgs  # noqa: E402
from paper_2506_12727_b200.dist import GradBuffer  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "garden"]
g_np, cams = synth.make_scene(cfg)
dev = torch.device("cuda", 0)
g = {k: torch.from_numpy(v).to(dev) for k, v in g_np.items() if isinstance(v, np.ndarray)}
g["sh_degree"] = g_np["sh_degree"]
dL = torch.from_numpy(synth.make_dLdC(cfg.V, cfg.H, cfg.W, cfg.seed)).to(dev)
R = mvgs.Rasterizer(0)
R.preprocess(g, cams)
st = R.stats
mvgs.reserve(R.ctx, int(st["Q"] * 1.15) + 4096, int(st["K"] * 1.15) + 65536)
outs = R.alloc_forward()
buf = GradBuffer(g_np["means"].shape[0], g_np["sh"].shape[1], dev)
mvgs.set_eval_counting(R.ctx, False)


def step():
    mvgs.preprocess(R.ctx, g, R.cams)
    mvgs.render_fwd(R.ctx, *outs)
    mvgs.render_bwd(R.ctx, dL, outs[1], outs[2])
    mvgs.adc_stats(R.ctx, buf.grads, buf.adc)


s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    for _ in range(3):
        step()
torch.cuda.current_stream().wait_stream(s)
torch.cuda.synchronize()
graph = torch.cuda.CUDAGraph()
with torch.cuda.graph(graph):
    step()
torch.cuda.synchronize()


def timed(fn, n=20):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


res = {"eager": [], "graph": []}
for _ in range(3):
    res["eager"].append(timed(step))
    res["graph"].append(timed(graph.replay))
print(json.dumps({"config": cfg.name, **{k: round(statistics.median(v), 4) for k, v in res.items()},
                  "all": res}), flush=True)
