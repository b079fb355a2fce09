#!/usr/bin/env python
"""bench_scaling.py — the 8-GPU strong-scaling argument of DESIGN.md §11, from single-GPU
measurements (this pool gives one GPU per call; `large`, 32 views split
over N GPUs, target ≥ 6× at N = 8).

Measured on one B200, CUDA events on the stream, median of --reps:
  t1            the whole 32-view step on one GPU (S1–S9);
  render(N)     rank 0's share: preprocess → render_fwd → render_bwd of its 32/N views;
  gauss_ar(N)   the all-reduce path's per-rank S8–S9: all P Gaussians over its 32/N views;
  owner(N)      the owner-sharded path's per-rank S8–S9: mvgs_owner_prepare (participation of
                its P/N Gaussians in all 32 views, slot layout, one host sync) + owner_adc_stats,
                fed with the slots every renderer would send it (replayed from one GPU that
                rendered all 32 views);
  bytes         all-reduce: the flat buffer, 4·(16 + 3·S)·P; owner: the largest number of
                slot bytes a rank sends or receives (48 B per slot, exact counts).
Model (stated assumptions): a ring/NVLS all-reduce moves 2(N−1)/N of the buffer at bus
bandwidth BW_ar and overlaps the per-Gaussian kernel of all but the last chunk; the owner
exchange moves its bytes point-to-point at BW_p2p per direction and is exposed.
  step_ar(N)    = render(N) + gauss_ar(N) + max(0, t_AR − gauss_ar(N)·(chunks−1)/chunks)
  step_owner(N) = render(N) + bytes_owner(N)/BW_p2p + owner(N)
  speedup       = t1 / step(N)
Prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402


def timed(fn, reps):
    import torch
    out = []
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b))
    return statistics.median(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="large")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--gpus", default="2,4,8")
    ap.add_argument("--bw-ar", type=float, default=700.0, help="assumed all-reduce bus bandwidth, GB/s")
    ap.add_argument("--bw-p2p", type=float, default=700.0, help="assumed point-to-point bandwidth per direction, GB/s")
    ap.add_argument("--chunks", type=int, default=4)
    args = ap.parse_args()
    import torch

    from paper_2506_12727_b200 import mvgs
    from paper_2506_12727_b200.dist import GradBuffer, exchange_plan, owner_bounds, view_renderer, view_shard

    cfg = synth.CONFIGS[args.config]
    g_np, cams = synth.make_scene(cfg)
    V, P, S = cfg.V, g_np["means"].shape[0], g_np["sh"].shape[1]
    dev = torch.device("cuda", 0)
    g = {k: torch.from_numpy(v).to(dev) for k, v in g_np.items() if isinstance(v, np.ndarray)}
    g["sh_degree"] = g_np["sh_degree"]
    dL = torch.from_numpy(synth.make_dLdC(V, cfg.H, cfg.W, cfg.seed)).to(dev)

    def ctx_for(c):
        R = mvgs.Rasterizer(0)
        R.preprocess(g, c)
        st = R.stats
        mvgs.reserve(R.ctx, int(st["Q"] * 1.15) + 4096, int(st["K"] * 1.15) + 65536)
        return R

    full = ctx_for(cams)
    fo = full.alloc_forward()
    buf = GradBuffer(P, S, dev)

    def step_full():
        mvgs.preprocess(full.ctx, g, cams)
        mvgs.render_fwd(full.ctx, *fo)
        mvgs.render_bwd(full.ctx, dL, fo[1], fo[2])
        mvgs.adc_stats(full.ctx, buf.grads, buf.adc)

    step_full()
    t1 = timed(step_full, args.reps)
    per_row = 16 + 3 * S
    ar_bytes = 4 * per_row * P
    res = {"config": f"{cfg.name}: {P} Gaussians SH{cfg.sh_degree}, {V} views at {cfg.W}x{cfg.H}",
           "t1_ms": round(t1, 3), "views_per_s_1gpu": round(V / (t1 / 1e3), 1), "allreduce_bytes": ar_bytes,
           "assumed": {"bw_allreduce_GBps": args.bw_ar, "bw_p2p_GBps": args.bw_p2p, "chunks": args.chunks},
           "per_N": {}}
    for N in [int(x) for x in args.gpus.split(",")]:
        lo, hi = view_shard(V, N, 0)
        cs = synth.subset_views(cams, lo, hi)
        R = ctx_for(cs)
        ro = R.alloc_forward()
        dLr = dL[lo:hi].contiguous()
        b = GradBuffer(P, S, dev)

        def render():
            mvgs.preprocess(R.ctx, g, cs)
            mvgs.render_fwd(R.ctx, *ro)
            mvgs.render_bwd(R.ctx, dLr, ro[1], ro[2])

        render()
        t_render = timed(render, args.reps)
        mvgs.adc_stats(R.ctx, b.grads, b.adc)
        t_gar = timed(lambda: mvgs.adc_stats(R.ctx, b.grads, b.adc), args.reps)
        # owner path: rank 0 owns bounds[0:1]; its slots of every view come from the full render
        step_full()
        bounds = owner_bounds(P, N)
        renderer = view_renderer(V, N)
        slot_off, slots = mvgs.owner_slices(full.ctx, bounds, V)
        # exact exchange volume: what each rank sends (its views' slices for other owners) / receives
        sent = np.zeros(N, np.int64)
        recv_n = np.zeros(N, np.int64)
        for v in range(V):
            r = renderer[v]
            for o in range(N):
                n = int(slot_off[v, o + 1] - slot_off[v, o])
                if o != r:
                    sent[r] += n
                    recv_n[o] += n
        owner_bytes = int(max(sent.max(), recv_n.max())) * 48
        ob = GradBuffer(int(bounds[1] - bounds[0]), S, dev)

        def owner():
            view_off, recv = mvgs.owner_prepare(full.ctx, cams, int(bounds[0]), int(bounds[1]))
            for v in range(V):  # what the renderers deliver (outside the timed S8–S9 in a real run)
                recv[view_off[v] * 12:view_off[v + 1] * 12].copy_(slots[slot_off[v, 0] * 12:slot_off[v, 1] * 12])
            return view_off

        owner()
        t_prep = timed(lambda: mvgs.owner_prepare(full.ctx, cams, int(bounds[0]), int(bounds[1])), args.reps)
        owner()
        t_og = timed(lambda: mvgs.owner_adc_stats(full.ctx, ob.grads, ob.adc), args.reps)
        t_ar = ar_bytes * 2 * (N - 1) / N / (args.bw_ar * 1e9) * 1e3
        exposed = max(0.0, t_ar - t_gar * (args.chunks - 1) / args.chunks)
        step_ar = t_render + t_gar + exposed
        t_x = owner_bytes / (args.bw_p2p * 1e9) * 1e3
        step_ow = t_render + t_x + t_prep + t_og
        res["per_N"][N] = {
            "views_per_rank": hi - lo, "render_ms": round(t_render, 3), "gauss_allreduce_path_ms": round(t_gar, 3),
            "allreduce_ms": round(t_ar, 3), "allreduce_exposed_ms": round(exposed, 3),
            "step_allreduce_ms": round(step_ar, 3), "speedup_allreduce": round(t1 / step_ar, 2),
            "owner_bytes_max_rank": owner_bytes, "owner_exchange_ms": round(t_x, 3),
            "owner_prepare_ms": round(t_prep, 3), "owner_gauss_ms": round(t_og, 3),
            "step_owner_ms": round(step_ow, 3), "speedup_owner": round(t1 / step_ow, 2)}
        del R
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
