"""Where the e2e step's time goes beyond the device-only step (garden, one GPU).

Times CUDA-graph replays of (a) the device step S1-S9, (b) the same plus the l1 loss kernel,
(c) (b) with the next step's 48.8 MB target upload running on a copy stream, (d) the upload
alone, and (e) the loss kernel alone.  Prints one JSON line.
  python scripts/e2e_probe.py [--config garden]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2506_12727_b200 import mvgs  # noqa: E402
from paper_2506_12727_b200.dist import GradBuffer  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="garden")
    ap.add_argument("--n", type=int, default=20)
    args = ap.parse_args()
    cfg = synth.CONFIGS[args.config]
    g_np, cams = synth.make_scene(cfg)
    dev = torch.device("cuda", 0)
    g = {k: torch.from_numpy(v).to(dev) for k, v in g_np.items() if isinstance(v, np.ndarray)}
    g["sh_degree"] = g_np["sh_degree"]
    R = mvgs.Rasterizer(0)
    R.preprocess(g, cams)
    st = R.stats
    mvgs.reserve(R.ctx, int(st["Q"] * 1.15) + 4096, int(st["K"] * 1.15) + 65536)
    mvgs.set_eval_counting(R.ctx, False)
    outs = R.alloc_forward()
    buf = GradBuffer(g_np["means"].shape[0], g_np["sh"].shape[1], dev)
    dL = torch.from_numpy(synth.make_dLdC(cfg.V, cfg.H, cfg.W, cfg.seed)).to(dev)
    host_tgt = torch.rand((cfg.V, 3, cfg.H, cfg.W)).pin_memory()
    tgt = host_tgt.to(dev)
    tgt2 = torch.empty_like(tgt)
    dLe = torch.empty_like(dL)
    loss = torch.zeros(1, dtype=torch.float64, device=dev)

    def device_step():
        mvgs.preprocess(R.ctx, g, R.cams)
        mvgs.render_fwd(R.ctx, *outs)
        mvgs.render_bwd(R.ctx, dL, outs[1], outs[2])
        mvgs.adc_stats(R.ctx, buf.grads, buf.adc)

    def e2e_compute():
        mvgs.preprocess(R.ctx, g, R.cams)
        mvgs.render_fwd(R.ctx, *outs)
        mvgs.loss_grad(R.ctx, outs[0], tgt, dLe, mode=mvgs.LOSS_L1, loss=loss)
        mvgs.render_bwd(R.ctx, dLe, outs[1], outs[2])
        mvgs.adc_stats(R.ctx, buf.grads, buf.adc)

    def loss_only():
        mvgs.loss_grad(R.ctx, outs[0], tgt, dLe, mode=mvgs.LOSS_L1, loss=loss)

    def capture(fn):
        fn()
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            fn()
        torch.cuda.synchronize()
        return gr

    gd, ge, gl = capture(device_step), capture(e2e_compute), capture(loss_only)
    cs = torch.cuda.Stream()

    def timed(fn, n):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(n):
            fn()
        z.record()
        torch.cuda.synchronize()
        return a.elapsed_time(z) / n

    def with_upload():
        with torch.cuda.stream(cs):
            tgt2.copy_(host_tgt, non_blocking=True)
        ge.replay()
        torch.cuda.current_stream().wait_stream(cs)

    def upload_only():
        tgt2.copy_(host_tgt, non_blocking=True)

    # the bench's e2e loop: double-buffered target slots and loss read-back, events between streams
    comp = torch.cuda.current_stream()
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    slots = [tgt, tgt2]
    losses = [loss, torch.zeros(1, dtype=torch.float64, device=dev)]
    loss_host = [torch.zeros(1, dtype=torch.float64).pin_memory() for _ in range(2)]
    mk = lambda: [torch.cuda.Event() for _ in range(2)]  # noqa: E731
    in_ready, in_free, out_ready, out_free = mk(), mk(), mk(), mk()

    def e2e_b(b):
        mvgs.preprocess(R.ctx, g, R.cams)
        mvgs.render_fwd(R.ctx, *outs)
        mvgs.loss_grad(R.ctx, outs[0], slots[b], dLe, mode=mvgs.LOSS_L1, loss=losses[b])
        mvgs.render_bwd(R.ctx, dLe, outs[1], outs[2])
        mvgs.adc_stats(R.ctx, buf.grads, buf.adc)

    gb = [capture(lambda: e2e_b(0)), capture(lambda: e2e_b(1))]

    def bench_loop(n, upload=True, readback=True):
        a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(comp)
        s_in.wait_event(a)
        for i in range(n):
            b = i % 2
            if upload:
                if i >= 2:
                    s_in.wait_event(in_free[b])
                with torch.cuda.stream(s_in):
                    slots[b].copy_(host_tgt, non_blocking=True)
                in_ready[b].record(s_in)
                comp.wait_event(in_ready[b])
            if readback and i >= 2:
                comp.wait_event(out_free[b])
            gb[b].replay()
            in_free[b].record(comp)
            if readback:
                out_ready[b].record(comp)
                s_out.wait_event(out_ready[b])
                with torch.cuda.stream(s_out):
                    loss_host[b].copy_(losses[b], non_blocking=True)
                out_free[b].record(s_out)
        if readback:
            comp.wait_event(out_free[(n - 1) % 2])
        z.record(comp)
        torch.cuda.synchronize()
        return a.elapsed_time(z) / n

    for up, rb in ((True, True), (True, True)):
        bench_loop(6, up, rb)
    loops = {f"loop_up{int(u)}_rb{int(r)}_ms": bench_loop(24, u, r) for u, r in
             ((True, True), (False, True), (True, False), (False, False))}

    out = {**loops,
        "config": args.config,
        "device_step_ms": timed(gd.replay, args.n),
        "e2e_compute_ms": timed(ge.replay, args.n),
        "e2e_compute_with_upload_ms": timed(with_upload, args.n),
        "upload_only_ms": timed(upload_only, args.n),
        "loss_only_ms": timed(gl.replay, args.n),
        "upload_bytes": host_tgt.numel() * 4,
    }
    print(json.dumps(out))


if __name__ == "__main__":
    main()
