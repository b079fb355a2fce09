#!/usr/bin/env python
"""bench_adc.py — NEXT-3: one multi-view ADC event (P:4) on B200.

Garden-scale input (3 M Gaussians, SH degree 3, synth.make_adc_inputs: ~7% split, ~8% cloned,
~4% pruned at B = 4) resident in HBM; times mvgs_adc_step (decide + scan + host read of the
new count + emit) with CUDA events, and reports the HBM roofline of the whole event from its
algorithmic bytes: per input Gaussian the decide pass reads log-scales,
opacity, two accumulators and denom (28 B) and writes count + flags (5 B); the emit pass reads
flags + offset + the full parameter row (5 + 236 B) and the split noise (24·N B per split
parent) and writes 241 B per output row (parameters + origin + kind).  The oracle is timed
on a bounded sample of parents for the cpu_baseline.  Prints one JSON line.
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
    ap.add_argument("--P", type=int, default=3_000_000)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--cpu-sample", type=int, default=100_000)
    args = ap.parse_args()
    import torch

    from paper_2506_12727_b200 import mvgs

    P, N = args.P, 2
    g, acc, noise = synth.make_adc_inputs(P, 11, N=N)
    cfg = dict(batch_views=4, prune_scale_max=0.1)
    gd = {k: torch.from_numpy(v).cuda() for k, v in g.items() if isinstance(v, np.ndarray)}
    gd["sh_degree"] = g["sh_degree"]
    ad = {("denom_acc" if k == "denom" else k + "_acc"): torch.from_numpy(v).cuda() for k, v in acc.items()}
    nz = torch.from_numpy(noise).cuda()
    cap = int(P * 1.6)
    out = mvgs.alloc_gaussians(cap, g["sh"].shape[1], "cuda")
    origin = torch.empty(cap, dtype=torch.int32, device="cuda")
    kind = torch.empty(cap, dtype=torch.uint8, device="cuda")
    ctx = mvgs.create(0)
    for _ in range(args.warmup):
        rep = mvgs.adc_step(ctx, gd, ad, nz, cfg, out, origin, kind)
    torch.cuda.synchronize()
    times = []
    for _ in range(args.steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rep = mvgs.adc_step(ctx, gd, ad, nz, cfg, out, origin, kind)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    ms = float(np.median(times))
    row = 12 + 12 + 16 + 4 + g["sh"].shape[1] * 12
    bytes_ = P * (28 + 5) + P * (5 + row) + rep["n_split"] * 24 * N + rep["P_new"] * (row + 5)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    hbm = None
    for k in ("hbm_gbs",):
        if k in peaks:
            hbm = float(peaks[k])
    if hbm is None:
        hbm = 6548.8
    achieved = bytes_ / (ms * 1e-3) / 1e9

    from oracle import adc as oadc
    idx = np.arange(min(args.cpu_sample, P))
    sub = lambda d: {k: (v[idx] if isinstance(v, np.ndarray) else v) for k, v in d.items()}  # noqa: E731
    t0 = time.perf_counter()
    oadc.adc_step(sub(g), sub(acc), noise[idx], oadc.default_config(**cfg))
    cpu_s = time.perf_counter() - t0
    line = {"metric": "multi-view ADC event time (NEXT-3)", "value": round(ms, 4), "unit": "ms/event",
            "higher_is_better": False, "steps": args.steps, "warmup": args.warmup, "dtype": "f32",
            "data": "synthetic (synth.make_adc_inputs)",
            "config": {"workload": f"{P} Gaussians SH3, N={N}, B=4", "report": rep},
            "gpu_launches": 5,
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                         "frac": round(achieved / hbm, 4), "algorithmic_bytes": int(bytes_),
                         "note": "whole event incl. the host read of the new count"},
            "cpu_baseline": {"value": round(cpu_s * P / len(idx) * 1e3, 1), "unit": "ms/event", "cores": 1,
                             "kind": "oracle", "sample": f"first {len(idx)} parents ({cpu_s:.2f} s), scaled to P"}}
    print(json.dumps(line), flush=True)
    mvgs.destroy(ctx)


if __name__ == "__main__":
    main()
