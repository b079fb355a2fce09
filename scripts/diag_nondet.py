"""Diagnostic: run-to-run spread of selected gradient elements (partial and full paths)."""
import sys
import numpy as np
import torch
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import synth  # noqa: E402
from gpu_harness import run_gpu, to_dev  # noqa: E402
from test_gpu_partial import dense_index, run_partial, sample_lists  # noqa: E402
from paper_2506_12727_b200 import mvgs  # noqa: E402

cfg = synth.scaled(synth.CONFIGS["garden"], P=20_000, V=4, W=203, H=137)
g, cams = synth.make_scene(cfg)
V, W, H = 4, 203, 137
TX, TY = (W + 15) // 16, (H + 15) // 16
pix = sample_lists(V, TX * TY, 64, 5)
v, y, x, inside = dense_index(pix, TX, H, W)
dL_full = synth.make_dLdC_scaled(V, H, W, 7)
dL_s = np.zeros(pix.shape + (3,), np.float32)
dL_s[inside] = dL_full[v[inside], :, y[inside], x[inside]]
vals = []
for it in range(8):
    out = run_partial(g, cams, pix, 0, dL_s)
    vals.append(out["d_means"].reshape(-1)[[32287, 33288]])
print("partial d_means[32287,33288] over runs:\n", np.array(vals))
# same pgrad, gauss_bwd twice: deterministic?
R = mvgs.Rasterizer(0)
R.preprocess(to_dev(g), cams)
dev = torch.device("cuda")
p = torch.from_numpy(pix).to(dev)
rgb = torch.empty((V, TX * TY, 64, 3), device=dev)
Tf = torch.empty((V, TX * TY, 64), device=dev)
nc = torch.empty((V, TX * TY, 64), dtype=torch.int32, device=dev)
mvgs.render_fwd_partial(R.ctx, p, 64, 0, rgb, Tf, nc)
mvgs.render_bwd_partial(R.ctx, p, 64, 0, torch.from_numpy(dL_s).to(dev), Tf, nc)
a = R.alloc_backward(); b = R.alloc_backward()
mvgs.adc_stats(R.ctx, *a); mvgs.adc_stats(R.ctx, *b)
torch.cuda.synchronize()
print("gauss_bwd twice on one pgrad equal:", all(torch.equal(a[0][k], b[0][k]) for k in a[0]))
# which pairs feed Gaussian 32287//3
gid = 32287 // 3
print("gid", gid, "d_means", a[0]["d_means"][gid].tolist())
Q = R.stats["Q"]
pid = torch.empty((Q, 2), dtype=torch.int32, device=dev); pi = torch.empty((Q, 8), dtype=torch.int32, device=dev)
pf = torch.empty((Q, 12), device=dev); pg = torch.empty((Q, 10), device=dev)
mvgs.export_pairs(R.ctx, pid, pi, pf, pg)
torch.cuda.synchronize()
sel = (pid[:, 1] == gid).nonzero().flatten().tolist()
for q in sel:
    print("pair", q, "view", pid[q, 0].item(), "rect", pi[q, 1:6].tolist(), "flags", pi[q, 6].item(), "grad", [round(t, 8) for t in pg[q].tolist()])
