#!/usr/bin/env python
"""bench_dssim.py — NEXT-2: the 3D distance-aware D-SSIM on B200.

Times mvgs_dssim3d (loss + ∂loss/∂img) on a garden-shaped batch (4 views of
1237×822, synthetic inputs from synth.make_dssim_inputs) with inputs resident in
HBM, per-kernel stage time from the library's event pairs, and the ALU roofline
of the two window kernels (flops per centre counted from the
kernel's arithmetic).  The oracle (oracle/dssim.py, fp64 numpy) is timed on a
bounded crop of one view for the cpu_baseline.  Prints one JSON line.
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

# flops per window centre, counted from k_dssim.cu:
#   centre kernel, per neighbour: 3D distance 8 + exp 4 + Σw 1 + 3 ch × (5 moments: 8) = 37; 121 neighbours;
#   epilogue ≈ 3 × 40.   grad kernel, per neighbour: distance 8 + exp 4 + scale 1 + 3 × 5 = 28.
FLOPS_CENTER = 121 * 37 + 120
FLOPS_GRAD = 121 * 28


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--V", type=int, default=4)
    ap.add_argument("--W", type=int, default=1237)
    ap.add_argument("--H", type=int, default=822)
    ap.add_argument("--cpu-crop", type=int, default=96)
    args = ap.parse_args()
    import torch

    from paper_2506_12727_b200 import mvgs

    V, H, W = args.V, args.H, args.W
    img, tgt, depth, Tf, cams = synth.make_dssim_inputs(V, H, W, seed=11)
    dev = torch.device("cuda", 0)
    t = [torch.from_numpy(a).to(dev) for a in (img, tgt, depth, Tf)]
    loss = torch.zeros(1, device=dev)
    g = torch.empty_like(t[0])
    ctx = mvgs.create(0)
    for _ in range(args.warmup):
        mvgs.dssim3d(ctx, cams, *t, loss, g)
    torch.cuda.synchronize()
    mvgs.set_timing(ctx, True)
    mvgs.stage_times(ctx)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        mvgs.dssim3d(ctx, cams, *t, loss, g)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    st = mvgs.stage_times(ctx)["dssim"]
    mvgs.set_timing(ctx, False)
    npx = V * H * W
    props = torch.cuda.get_device_properties(0)
    try:
        import pynvml
        pynvml.nvmlInit()
        sm_max = pynvml.nvmlDeviceGetMaxClockInfo(pynvml.nvmlDeviceGetHandleByIndex(0), pynvml.NVML_CLOCK_SM)
    except Exception:
        sm_max = 1965
    peak = props.multi_processor_count * 128 * 2 * sm_max * 1e6 / 1e12
    achieved = npx * (FLOPS_CENTER + FLOPS_GRAD) / (st * 1e-3) / 1e12

    # cpu baseline: the oracle on a crop of one view
    c = args.cpu_crop
    from oracle import dssim
    t0 = time.perf_counter()
    dssim.dssim3d(img[:1, :, :c, :c], tgt[:1, :, :c, :c], depth[:1, :c, :c], Tf[:1, :c, :c], cams[:1])
    cpu_s = time.perf_counter() - t0
    line = {"metric": "3D D-SSIM loss+grad throughput (NEXT-2)", "value": round(V / (ms * 1e-3), 2),
            "unit": "views/s", "ms_per_step": round(ms, 4), "steps": args.steps, "warmup": args.warmup,
            "dtype": "f32", "data": "synthetic (synth.make_dssim_inputs)",
            "config": {"workload": f"{V} views {W}x{H}, 11x11 windows, sigma_px 1.5"},
            "gpu_launches": 3 * ((V + 63) // 64) if V <= 64 else None,
            "roofline": {"bound": "alu", "achieved": round(achieved, 3), "peak": round(peak, 2), "unit": "TFLOP/s",
                         "frac": round(achieved / peak, 4), "kernel": "dssim (center+grad)",
                         "flops_per_px": FLOPS_CENTER + FLOPS_GRAD, "stage_ms": round(st, 4)},
            "cpu_baseline": {"value": round((c * c) / (H * W) / cpu_s, 5), "unit": "views/s", "cores": 1,
                             "kind": "oracle", "sample": f"one {c}x{c} crop of view 0 ({cpu_s:.2f} s)"}}
    print(json.dumps(line), flush=True)
    mvgs.destroy(ctx)


if __name__ == "__main__":
    main()
