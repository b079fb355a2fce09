#!/usr/bin/env python
"""bench_variance.py — NEXT-4: a synthetic analog of Fig. 3 on B200.

Frozen garden-shaped scene (3 M Gaussians, SH 3, 1237×822), M = 16 views orbiting it with
seeded target photos (synth.make_lab_targets).  For B ∈ {1, 2, 4, 8} views per mini-batch,
K seeded batches of B distinct views are drawn; each batch's ∂L/∂means (ℓ2 loss) goes through
the full S1–S8 path and the §4.2 estimator runs on the GPU.  Also computes the
population variance σ² of the M single-view gradients (every view once) and the textbook
without-replacement prediction 𝕍(B) = σ²/B·(M − B)/(M − 1) that the estimates should follow.
Reports batch-gradient throughput at each B.  Prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--M", type=int, default=16)
    ap.add_argument("--K", type=int, default=48)
    ap.add_argument("--config", default="garden")
    args = ap.parse_args()
    import torch

    from paper_2506_12727_b200 import mvgs
    from paper_2506_12727_b200.lab import VarianceLab

    cfg = synth.scaled(synth.CONFIGS[args.config], V=args.M)
    g_np, cams = synth.make_scene(cfg)
    dev = torch.device("cuda", 0)
    g = {k: torch.from_numpy(v).to(dev) for k, v in g_np.items() if isinstance(v, np.ndarray)}
    g["sh_degree"] = g_np["sh_degree"]
    targets = torch.from_numpy(synth.make_lab_targets(args.M, cfg.H, cfg.W, cfg.seed)).to(dev)
    lab = VarianceLab(g, cams, targets, loss=mvgs.LOSS_L2)
    # size the context once (largest batch), then run without per-batch host syncs
    lab.batch_gradient(list(range(8)))
    st = lab.R.stats
    mvgs.reserve(lab.R.ctx, int(st["Q"] * 1.3) + 4096, int(st["K"] * 1.3) + 65536)
    lab.auto_reserve = False
    sigma2 = lab.run([[i] for i in range(args.M)])  # population variance of the per-view gradients
    rng = np.random.default_rng(cfg.seed)
    rows = []
    for B in (1, 2, 4, 8):
        batches = [list(rng.choice(args.M, B, replace=False)) for _ in range(args.K)]
        lab.run(batches[:2])  # warm the per-B buffers
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        v = lab.run(batches)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        pred = sigma2 / B * (args.M - B) / (args.M - 1)
        rows.append({"B": B, "variance": v, "predicted": pred, "ratio_to_B1": None,
                     "batch_grads_per_s": round(args.K / (ms * 1e-3), 2),
                     "views_per_s": round(args.K * B / (ms * 1e-3), 2), "wall_s": round(time.perf_counter() - t0, 3)})
    for r in rows:
        r["ratio_to_B1"] = round(r["variance"] / rows[0]["variance"], 4)
    line = {"metric": "Fig. 3 analog: mini-batch gradient variance vs views per batch (NEXT-4)",
            "unit": "variance of ∂L/∂means (ℓ2 loss), fp64",
            "config": {"workload": f"{cfg.name}: {cfg.P} Gaussians SH{cfg.sh_degree}, M={args.M} views "
                                   f"{cfg.W}x{cfg.H}, K={args.K} batches per B, frozen parameters"},
            "sigma2_population": sigma2, "rows": rows,
            "paper_context": "Fig. 3: single-view mini-batches show larger gradient variance than multi-view (P:157-160)"}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
