#!/usr/bin/env python
"""bench_partial.py — NEXT-1: the Table 4 speed analog on B200.

Per iteration, the multi-view step on the garden-shaped batch (3 M Gaussians,
SH 3, 4 views of 1237×822) in three ways:
  full        every pixel of the 4 views (bench.py's step);
  masked      each (view, tile) renders S = 256/4 sub-sampled pixels with a
              256-thread block and the rest masked off (the paper's "Partial",
              P:314);
  efficient   the same pixels with ⌈S/32⌉·32-thread blocks (Alg. 3).
Masked and efficient render one image's worth of pixels per iteration.
Prints one JSON line: ms per step and per compositing stage for each arm.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="garden")
    args = ap.parse_args()
    import torch

    from paper_2506_12727_b200 import mvgs
    from paper_2506_12727_b200.dist import GradBuffer

    cfg = synth.CONFIGS[args.config]
    g_np, cams = synth.make_scene(cfg)
    dev = torch.device("cuda", 0)
    g = {k: torch.from_numpy(v).to(dev) for k, v in g_np.items() if isinstance(v, np.ndarray)}
    g["sh_degree"] = g_np["sh_degree"]
    V, H, W = cfg.V, cfg.H, cfg.W
    TX, TY = (W + 15) // 16, (H + 15) // 16
    T = TX * TY
    S = 256 // V
    rng = np.random.default_rng(cfg.seed)
    pix = torch.from_numpy(np.stack([np.stack([rng.choice(256, S, replace=False) for _ in range(T)])
                                     for _ in range(V)]).astype(np.int32)).to(dev)
    dL_full = torch.from_numpy(synth.make_dLdC(V, H, W, cfg.seed)).to(dev)
    dL_s = torch.from_numpy((np.random.default_rng(1).integers(0, 2, (V, T, S, 3)) * 2.0 - 1.0).astype(np.float32)
                            / np.float32(3 * V * T * S)).to(dev)
    R = mvgs.Rasterizer(0)
    R.preprocess(g, cams)
    st = R.stats
    mvgs.reserve(R.ctx, int(st["Q"] * 1.15) + 4096, int(st["K"] * 1.15) + 65536)
    buf = GradBuffer(g_np["means"].shape[0], g_np["sh"].shape[1], dev)
    full_out = R.alloc_forward()
    p_rgb = torch.empty((V, T, S, 3), device=dev)
    p_T = torch.empty((V, T, S), device=dev)
    p_n = torch.empty((V, T, S), dtype=torch.int32, device=dev)

    def step(arm):
        mvgs.preprocess(R.ctx, g, R.cams)
        if arm == "full":
            mvgs.render_fwd(R.ctx, *full_out)
            mvgs.render_bwd(R.ctx, dL_full, full_out[1], full_out[2])
        else:
            mode = mvgs.PARTIAL_MASKED if arm == "masked" else mvgs.PARTIAL_THREAD_EFFICIENT
            mvgs.render_fwd_partial(R.ctx, pix, S, mode, p_rgb, p_T, p_n)
            mvgs.render_bwd_partial(R.ctx, pix, S, mode, dL_s, p_T, p_n)
        mvgs.adc_stats(R.ctx, buf.grads, buf.adc)

    res = {}
    for arm in ("full", "masked", "efficient"):
        for _ in range(args.warmup):
            step(arm)
        torch.cuda.synchronize()
        mvgs.set_timing(R.ctx, True)
        mvgs.stage_times(R.ctx)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            step(arm)
        e1.record()
        torch.cuda.synchronize()
        stages = mvgs.stage_times(R.ctx)
        mvgs.set_timing(R.ctx, False)
        ms = e0.elapsed_time(e1) / args.steps
        px = V * H * W if arm == "full" else int((p_n.numel()))
        res[arm] = {"ms_per_step": round(ms, 4), "fwd_ms": round(stages["render_fwd"], 4),
                    "bwd_ms": round(stages["render_bwd"], 4), "pixels_per_step": px,
                    "views_per_s": round(V / (ms / 1e3), 2)}
        # occupancy: threads holding a pixel / threads launched, and lane-steps
        # of the entry walk spent on a live pixel / executed (the kernels count them)
        if arm == "full":  # 256 pixel slots per (view, tile) CTA (128 threads × 2 pixels)
            res[arm]["occupancy_threads"] = round(V * H * W / (V * T * 256), 4)
        else:
            st = mvgs.query(R.ctx)
            res[arm]["threads_launched"] = st["threads_launched"]
            res[arm]["threads_active"] = st["threads_active"]
            res[arm]["occupancy_threads"] = round(st["threads_active"] / max(1, st["threads_launched"]), 4)
            res[arm]["occupancy_lane_steps"] = round(st["lane_steps_active"] / max(1, st["lane_steps_launched"]), 4)
    line = {"metric": "Table-4 analog: multi-view step time, full vs masked-partial vs thread-efficient-partial",
            "unit": "ms/step", "config": {"workload": f"{cfg.name}: {cfg.P} Gaussians SH{cfg.sh_degree}, {V} views "
                                                      f"{W}x{H}, S={S} sampled pixels per (view, tile)"},
            "arms": res,
            "paper_context": "Table 4 (RTX 3090, whole training): Full 127 min, Partial 105 min, Ours 50 min (P:262-264)",
            "speedup_efficient_vs_full_render": round((res["full"]["fwd_ms"] + res["full"]["bwd_ms"])
                                                      / (res["efficient"]["fwd_ms"] + res["efficient"]["bwd_ms"]), 3),
            "speedup_efficient_vs_masked_render": round((res["masked"]["fwd_ms"] + res["masked"]["bwd_ms"])
                                                        / (res["efficient"]["fwd_ms"] + res["efficient"]["bwd_ms"]), 3)}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
