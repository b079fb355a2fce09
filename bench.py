#!/usr/bin/env python
"""bench.py — views/s of the batched multi-view rasterizer step on B200.

One step = the whole hot path on one batch:
preprocess (S1–S5) → render_fwd (S6) → render_bwd (S7) → adc_stats (S8–S9),
plus, with N > 1 GPUs, the NCCL all-reduce of the flat [param grads | E1 | E2 | vis]
buffer (every output is a sum over views), issued per Gaussian chunk
as soon as that chunk's S8–S9 kernel is enqueued (MVGS_AR_CHUNKS, default 4) so the
collective overlaps the rest of the per-Gaussian kernel.

Workload: BASELINE.json configs[1], the Mip-NeRF-360 garden-shaped scene
(3 M Gaussians, SH degree 3, 4 views of 1237×822) per GPU; with N GPUs each rank
renders its own 4 views of the same scene (4·N views, weak scaling).  Inputs are
resident in HBM and larger than L2 (708 MB of parameters).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config garden]
  python bench.py --impl reference      # the oracle (CPU) on a bounded sample

Prints ONE JSON line (rank 0).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "views/sec fwd+bwd (N-view batch, 1/2/4/8 B200) and % HBM/L2 roofline"
UNIT = "views/s"

# fp32 flops of one (pixel, entry) evaluation, counted from the CA forms of
# DESIGN.md §4 (FMA = 2): every evaluation pays the offset + power + skip test
# (13); those above the exact skip bound also pay the rest
FLOPS_VISIT = 13
FWD_FLOPS_REST = 29
BWD_FLOPS_REST = 83


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="garden", choices=list(synth.CONFIGS))
    ap.add_argument("--views", type=int, default=0,
                    help="views per GPU per step (default: the config's batch); the views-per-batch sweep")
    ap.add_argument("--impl", default="mvgs", choices=["mvgs", "reference"])
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: the config's batch per GPU; strong: the config's batch split over the GPUs "
                         "(SURVEY §8(d): large, 32 views)")
    ap.add_argument("--exchange", default="allreduce", choices=["allreduce", "owner"],
                    help="N>1 exchange: chunked all-reduce of the flat buffer, or owner-sharded slots (DESIGN §11)")
    ap.add_argument("--e2e-steps", type=int, default=24)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--eager", action="store_true", help="time eager launches instead of one CUDA-graph replay per step")
    ap.add_argument("--profile", action="store_true",
                    help="sizing pass + warmup + one step, nothing else (for ncu)")
    return ap.parse_args()


# --------------------------------------------------------------------- clocks
class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        rows = []
        for line in open(self.f.name):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[j] for r in rows for j in range(4) if r[5 + j].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# --------------------------------------------------------------- distributed
def dist_setup():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured"
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


def measured_alu_peak():
    """FFMA2 TFLOP/s measured on a B200 of this pool (scripts/microbench_alu.cu), or None."""
    try:
        return float(json.load(open(os.path.join(ROOT, "profiles", "r2_alu_peaks.json")))["ffma2_tflops"])
    except (OSError, ValueError, KeyError):
        try:  # the file holds one JSON object per line (two runs)
            return float(json.loads(open(os.path.join(ROOT, "profiles", "r2_alu_peaks.json")).readline())["ffma2_tflops"])
        except (OSError, ValueError, KeyError):
            return None


def stage_models(P, NK, V, NB, Q, K, T, evf, evb, exf, exb, Qv):
    """(bound, algorithmic units per launch) per stage — DESIGN.md §7.  Qv = pairs with
    tiles > 0 (the rest are inert: only their depth, flags and sort key are written)."""
    pbytes = 4 * (11 + 3 * NK) * P
    return {
        "count": ("hbm", 24 * P + (4 * P if V <= 32 else 0) + 4 * V * NB),  # means + log_scales in, pmask out
        "scan_pairs": ("hbm", 3 * 4 * V * NB),
        "project": ("hbm", pbytes + 4 * V * NB + Qv * (48 + 4 + 4 + 8) + (Q - Qv) * (16 + 4 + 4)),
        "scan_buckets": ("hbm", 3 * 4 * V * T),
        "sort_pairs": ("hbm", 4 * 16 * Q),
        "dup": ("hbm", Q * (4 + 16 + 8 + 4 + 4) + 8 * K),
        "sort_entries": ("hbm", ((max(1, (V * T - 1).bit_length()) + 7) // 8) * 16 * K),
        "render_fwd": ("alu", FLOPS_VISIT * evf + FWD_FLOPS_REST * exf),
        "render_bwd": ("alu", FLOPS_VISIT * evb + BWD_FLOPS_REST * exb),
        "gauss_bwd": ("hbm", 2 * pbytes + 4 * Q + 48 * Qv + 16 * P),
    }


def launches_per_step(nbuckets, Q, K):
    """Kernels libmvgs launches per step: count + scan, project,
    pair sort (upsweep + bases + 4 onesweep passes; the last also writes the tile counts), scan + dup,
    entry sort (⌈log2(V·T)/8⌉ passes × (histogram + scan + scatter)),
    (the first pass's histogram is counted by dup), ranges close-up (segment minima + close;
    the bucket starts come out of the last entry pass), fwd, bwd, gauss_bwd."""
    ent_passes = (max(1, (nbuckets - 1).bit_length()) + 7) // 8
    return (1 + 1) + 1 + (2 + 4) + (1 + 1) + (3 * ent_passes - 1) + 2 + 3  # scans: one kernel each


# ---------------------------------------------------------------------- mvgs
def run_mvgs(args):
    import torch

    ws, rank, local = dist_setup()
    N = args.gpus if ws == 1 else ws
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2506_12727_b200 import mvgs
    from paper_2506_12727_b200.dist import GradBuffer, adc_stats_allreduce, adc_stats_owner, owner_bounds, view_shard

    cfg = synth.CONFIGS[args.config]
    if args.scaling == "weak":  # the per-GPU batch is fixed
        V_all = (args.views or cfg.V) * N
    else:  # strong: the batch is fixed and split over the GPUs
        V_all = args.views or cfg.V
    g_np, cams_all = synth.make_scene(synth.scaled(cfg, V=V_all))
    lo, hi = view_shard(V_all, N, rank)
    Vr = hi - lo
    cams = synth.subset_views(cams_all, lo, hi)
    P = g_np["means"].shape[0]
    NK = (g_np["sh_degree"] + 1) ** 2
    S = g_np["sh"].shape[1]
    dev = torch.device("cuda", local)
    g = {k: torch.from_numpy(v).to(dev) for k, v in g_np.items() if isinstance(v, np.ndarray)}
    g["sh_degree"] = g_np["sh_degree"]
    dL = torch.from_numpy(synth.make_dLdC(Vr, cfg.H, cfg.W, cfg.seed + rank)).to(dev)

    R = mvgs.Rasterizer(local)
    R.preprocess(g, cams)  # sizes the workspace (query + reserve), untimed
    st0 = R.stats
    mvgs.reserve(R.ctx, int(st0["Q"] * 1.15) + 4096, int(st0["K"] * 1.15) + 65536)
    # one flat buffer for every output that is a sum over views (single all-reduce)
    # with N > 1, chunk-major so each chunk's all-reduce overlaps the next chunk's kernel
    CHUNKS = int(os.environ.get("MVGS_AR_CHUNKS", "4")) if (dist is not None and args.exchange == "allreduce") else 1
    owner = args.exchange == "owner"
    if owner:  # this rank's outputs: the full sums of the Gaussians it owns (reduce-scatter semantics)
        ob = owner_bounds(P, N)
        buf = GradBuffer(int(ob[rank + 1] - ob[rank]), S, dev)
    else:
        buf = GradBuffer(P, S, dev, chunks=CHUNKS)
    flat = buf.flat
    outs = R.alloc_forward()

    checked = [False]  # the first (warm-up) exchange verifies every slice size across ranks

    def grads_out(b):
        mvgs.render_bwd(R.ctx, dL_cur[0], outs[1], outs[2])
        adc_out(b)

    def adc_out(b):  # S8–S9 (+ the exchange when N > 1)
        if owner:
            adc_stats_owner(R.ctx, P, cams_all, rank, N, b.grads, b.adc, check=not checked[0])
            checked[0] = True
        elif dist is None:
            mvgs.adc_stats(R.ctx, b.grads, b.adc)
        else:
            adc_stats_allreduce(R.ctx, b)

    dL_cur = [dL]

    def step():
        mvgs.preprocess(R.ctx, g, R.cams)
        mvgs.render_fwd(R.ctx, *outs)
        grads_out(buf)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if args.profile:  # the profiled step is bracketed for `ncu --profile-from-start off`
        if os.environ.get("MVGS_BENCH_COUNT", "0") != "1":
            mvgs.set_eval_counting(R.ctx, False)  # the timed steps' kernel variants
        step()
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        step()
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        print(json.dumps({"profile": True, "stats": mvgs.query(R.ctx)}), flush=True)
        return
    st = mvgs.query(R.ctx)  # structural stats of this workload incl. evaluation counts (sync, untimed)
    if os.environ.get("MVGS_BENCH_COUNT", "0") != "1":
        mvgs.set_eval_counting(R.ctx, False)  # statistics off in the timed steps (same workload, same counts)
    # One GPU: the step (S1–S9, every kernel) is captured once into a CUDA graph and replayed —
    # the launch-bound tail of a 27-launch step.  Several GPUs: eager steps (the
    # all-reduce chunks / owner exchange stay outside capture).
    graph = None
    if dist is None and not owner and not args.eager:
        cs = torch.cuda.Stream()
        cs.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(cs):
            step()
        torch.cuda.current_stream().wait_stream(cs)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
        torch.cuda.synchronize()
        for _ in range(args.warmup):
            graph.replay()
        torch.cuda.synchronize()
    run_step = graph.replay if graph is not None else step
    clk = Clocks(local)
    clk.start()
    time.sleep(0.3)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]  # per-step distribution
    ev0.record()
    evs[0].record()
    for i in range(args.steps):
        run_step()
        evs[i + 1].record()
    ev1.record()
    torch.cuda.synchronize()
    per_step = sorted(evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps))
    pct = lambda q: per_step[min(len(per_step) - 1, int(round(q * (len(per_step) - 1))))]  # noqa: E731
    if dist is not None:
        dist.barrier()
    clocks = clk.stop()
    ms = ev0.elapsed_time(ev1) / args.steps
    # Per-stage kernel times: a second timed region of the same K steps, eager, with a pair of
    # CUDA events around every stage on the launching stream (events between kernels add
    # ≈ 2 % of idle gaps, so the headline region above carries none).
    mvgs.set_timing(R.ctx, True)
    mvgs.stage_times(R.ctx)  # clear
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    es0, es1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    es0.record()
    for i in range(args.steps):
        step()
    es1.record()
    torch.cuda.synchronize()
    ms_staged = es0.elapsed_time(es1) / args.steps
    stages = mvgs.stage_times(R.ctx)
    mvgs.set_timing(R.ctx, False)
    if dist is not None:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    views_total = V_all
    value = views_total / (ms / 1e3)

    # ---- e2e: the step as a training iteration drives it through the public API, with HOST
    # buffers.  Every step uploads that step's inputs — the V target images (pinned host, the
    # photographs of the batch's views) — renders, forms the ℓ1 loss and its per-pixel
    # gradient on the device (mvgs_loss_grad), runs the backward and S8–S9, and reads the
    # loss back to the host.  The Gaussians stay resident (they are the model, updated on the
    # device between steps); targets are double-buffered, so step i+1's upload overlaps step i.
    # Timed from the first upload to the last loss read on the device.
    #   (e2e.host_resident_params: the same with the whole parameter set uploaded and the whole
    #   gradient + ADC buffer downloaded every step — a model kept in host memory.)
    rng_t = np.random.default_rng(cfg.seed + 7)
    # 8-bit target images, as photographs are stored (mvgs_loss_grad_u8 reads t/255): 1 B per value
    host_tgt = torch.from_numpy(rng_t.integers(0, 256, (Vr, 3, cfg.H, cfg.W), dtype=np.uint8)).pin_memory()
    tgt_slots = [torch.empty_like(host_tgt, device=dev) for _ in range(2)]
    loss_dev = [torch.zeros(1, dtype=torch.float64, device=dev) for _ in range(2)]
    loss_host = [torch.zeros(1, dtype=torch.float64).pin_memory() for _ in range(2)]
    comp = torch.cuda.current_stream()
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    mk = lambda: [torch.cuda.Event() for _ in range(2)]  # noqa: E731
    in_ready, in_free, out_ready, out_free = mk(), mk(), mk(), mk()
    h2d = host_tgt.numel() * host_tgt.element_size()
    d2h = 8

    def e2e_compute(b):  # the device part of one training iteration (slot b's target and loss)
        mvgs.preprocess(R.ctx, g, R.cams)
        mvgs.render_fwd(R.ctx, *outs)
        # the ℓ1 loss of the 8-bit targets fused into S7 (∂L/∂C formed per pixel in the backward)
        mvgs.render_bwd_l1(R.ctx, outs[0], tgt_slots[b], outs[1], outs[2], loss=loss_dev[b])
        adc_out(buf)

    # One GPU: each slot's compute is one CUDA graph (as the device-only step), replayed on the
    # compute stream between the event waits of the copy streams.
    e2e_graphs = [None, None]
    if graph is not None:
        for b in range(2):
            e2e_compute(b)  # warm (outside capture)
            torch.cuda.synchronize()
            e2e_graphs[b] = torch.cuda.CUDAGraph()
            with torch.cuda.graph(e2e_graphs[b]):
                e2e_compute(b)
            torch.cuda.synchronize()

    def e2e_step(i):
        b = i % 2
        if i >= 2:
            s_in.wait_event(in_free[b])
        with torch.cuda.stream(s_in):
            tgt_slots[b].copy_(host_tgt, non_blocking=True)
        in_ready[b].record(s_in)
        comp.wait_event(in_ready[b])
        if i >= 2:
            comp.wait_event(out_free[b])
        if e2e_graphs[b] is not None:
            e2e_graphs[b].replay()
        else:
            e2e_compute(b)
        in_free[b].record(comp)
        out_ready[b].record(comp)
        s_out.wait_event(out_ready[b])
        with torch.cuda.stream(s_out):
            loss_host[b].copy_(loss_dev[b], non_blocking=True)
        out_free[b].record(s_out)

    def e2e_time(step_fn, n):
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(comp)
        s_in.wait_event(a)
        for i in range(n):
            step_fn(i)
        comp.wait_event(out_free[(n - 1) % 2])
        z.record(comp)
        torch.cuda.synchronize()
        t = a.elapsed_time(z) / n
        if dist is not None:
            tt = torch.tensor([t], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t = float(tt.item())
        return t

    for i in range(6):  # warm-up: the pinned buffers' first transfers run slower
        e2e_step(i)
    e2e_ms = e2e_time(e2e_step, args.e2e_steps)

    # host-resident parameters: whole parameter set up, whole output buffer down, every step
    host_in = {k: torch.from_numpy(v).pin_memory() for k, v in g_np.items() if isinstance(v, np.ndarray)}
    host_dL = dL.cpu().pin_memory()
    host_out = [torch.empty_like(flat, device="cpu").pin_memory() for _ in range(2)]
    h2d_full = sum(t.numel() * 4 for t in host_in.values()) + host_dL.numel() * 4
    d2h_full = host_out[0].numel() * 4
    g_slots = [g, {k: (torch.empty_like(v) if torch.is_tensor(v) else v) for k, v in g.items()}]
    dL_slots = [dL, torch.empty_like(dL)]
    bufs = [buf, GradBuffer(buf.P, S, dev, chunks=CHUNKS)]

    def e2e_full_step(i):
        b = i % 2
        if i >= 2:
            s_in.wait_event(in_free[b])
        with torch.cuda.stream(s_in):
            for k, t in host_in.items():
                g_slots[b][k].copy_(t, non_blocking=True)
            dL_slots[b].copy_(host_dL, non_blocking=True)
        in_ready[b].record(s_in)
        comp.wait_event(in_ready[b])
        if i >= 2:
            comp.wait_event(out_free[b])
        ob = bufs[b]
        mvgs.preprocess(R.ctx, g_slots[b], R.cams)
        mvgs.render_fwd(R.ctx, *outs)
        dL_cur[0] = dL_slots[b]
        grads_out(ob)
        in_free[b].record(comp)
        out_ready[b].record(comp)
        s_out.wait_event(out_ready[b])
        with torch.cuda.stream(s_out):
            host_out[b].copy_(ob.flat, non_blocking=True)
        out_free[b].record(s_out)

    e2e_full_ms = e2e_time(e2e_full_step, max(4, args.e2e_steps // 2))
    dL_cur[0] = dL

    # ---- roofline of the dominant kernel
    peaks, peak_src = measured_peaks()
    T = st["tiles_x"] * st["tiles_y"]
    NB = (P + 255) // 256
    models = stage_models(P, NK, Vr, NB, st["Q"], st["K"], T, st["eval_fwd"], st["eval_bwd"], st["exp_fwd"],
                          st["exp_bwd"], st["n_visible"])
    dom = max(stages, key=lambda k: stages[k])
    bound, units = models[dom]
    t_dom = stages[dom] / 1e3
    if bound == "hbm":
        achieved = units / t_dom / 1e9
        peak = float(peaks["hbm_gbs"])
        unit = "GB/s"
    else:
        achieved = units / t_dom / 1e12
        peak = 148 * 128 * 2 * float(peaks.get("sm_max_mhz", 1965.0)) * 1e6 / 1e12
        unit = "TFLOP/s"
    traffic = None
    tp = os.path.join(ROOT, "profiles", f"traffic_{args.config}.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get(dom)
    roof = {"bound": bound, "achieved": round(achieved, 3), "peak": round(peak, 3), "unit": unit,
            "frac": round(achieved / peak, 4), "traffic": traffic, "kernel": dom,
            "peak_source": peak_src if bound == "hbm" else "derived: 148 SM x 128 FP32 lanes x 2 x sm_max_mhz",
            **({} if bound == "hbm" else {"peak_measured": measured_alu_peak()}),
            "stage_ms": {k: round(v, 4) for k, v in stages.items()},
            "stage_frac": {k: round(models[k][1] / (stages[k] / 1e3) / (1e9 * float(peaks["hbm_gbs"]) if models[k][0] == "hbm" else peak * 1e12), 4)
                           for k in stages if stages[k] > 0}}

    line = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": N, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 4),
        "step_ms_p10_p50_p90": [round(pct(0.1), 4), round(pct(0.5), 4), round(pct(0.9), 4)],
        "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (mvgs-synth v1, seeded; DESIGN.md §6)",
        "config": {**workload_config(cfg, P, Vr, N, V_all),
                   "exchange": args.exchange if N > 1 or owner else "none (1 GPU)",
                   "allreduce_chunks": CHUNKS,
                   "launch": "CUDA graph replay (one capture of S1-S9)" if graph is not None else "eager",
                   "stage_timing": "second region of %d eager steps with events around each stage: %.4f ms/step"
                                   % (args.steps, ms_staged),
                   "l2": "inputs larger than L2 (params %.0f MB)" % (sum(v.nbytes for v in g_np.values()
                                                                       if isinstance(v, np.ndarray)) / 1e6),
                   "Q": st["Q"], "K": st["K"], "max_bucket": st["max_bucket"], "n_visible": st["n_visible"],
                   # structural statistics: ρ = Q/(V·P), κ = K/Q_visible, mean list length
                   "rho": round(st["Q"] / max(1, Vr * P), 4), "kappa": round(st["K"] / max(1, st["n_visible"]), 3),
                   "mean_bucket": round(st["K"] / max(1, Vr * st["tiles_x"] * st["tiles_y"]), 1),
                   "eval_fwd_per_px": round(st["eval_fwd"] / (Vr * cfg.W * cfg.H), 2),
                   "eval_bwd_per_px": round(st["eval_bwd"] / (Vr * cfg.W * cfg.H), 2),
                   "exp_fwd_per_px": round(st["exp_fwd"] / (Vr * cfg.W * cfg.H), 2),
                   "exp_bwd_per_px": round(st["exp_bwd"] / (Vr * cfg.W * cfg.H), 2)},
        "clocks": clocks,
        "e2e": {"value": round(views_total / (e2e_ms / 1e3), 3), "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": round(e2e_ms, 3),
                "step": "8-bit target images up (pinned, double-buffered), render, backward with the l1 loss and "
                        "dL/dC fused in (mvgs_render_bwd_l1) + S8-S9, loss down; Gaussians resident",
                "launch": ("compute of each step one CUDA graph replay (per target slot); copies and "
                           "event waits eager" if e2e_graphs[0] is not None else "eager"),
                "host_resident_params": {"value": round(views_total / (e2e_full_ms / 1e3), 3), "unit": UNIT,
                                         "h2d_bytes_per_step": h2d_full, "d2h_bytes_per_step": d2h_full,
                                         "ms_per_step": round(e2e_full_ms, 3)}},
        "gpu_launches": launches_per_step(Vr * T, st["Q"], st["K"]) * args.steps,
        "roofline": roof,
    }
    if rank == 0 and N == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, g_np, cams, dL.cpu().numpy())
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


# ---------------------------------------------------------------- oracle arm
def host_cpu():
    """(logical cores, model name) of this host (the GPU box's, when run there)."""
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return os.cpu_count() or 1, model


def oracle_threads():
    """All host cores (SURVEY §8(d) M6 oracle-mt), capped at 64 (per-thread pair accumulators)."""
    return max(1, min(64, int(os.environ.get("MVGS_ORACLE_THREADS", os.cpu_count() or 1))))


def oracle_sample(g_np, cams, dL, frac, seed=0, threads=1):
    """Time the oracle (the C oracle as it stands, on `threads` host threads: OpenMP over
    Gaussians and (view, tile) buckets) on a bounded sample of the workload: view 0 with a
    seeded fraction `frac` of its 16×16 tiles (∂L/∂C zero elsewhere), all stages S1–S9.
    Returns (views/s = frac / seconds, seconds, sample)."""
    import oracle
    oracle.set_threads(threads)
    W, H = int(cams[0]["width"]), int(cams[0]["height"])
    TX, TY = (W + 15) // 16, (H + 15) // 16
    T = TX * TY
    mask = None
    d = dL[:1]
    nt = T
    if frac < 1.0:
        rng = np.random.default_rng(seed)
        nt = max(1, int(round(frac * T)))
        m = np.zeros(T, np.uint8)
        m[rng.choice(T, nt, replace=False)] = 1
        mask = m.reshape(1, T)
        pix = np.repeat(np.repeat(m.reshape(TY, TX), 16, 0), 16, 1)[:H, :W].astype(bool)
        d = dL[:1] * pix[None, None]
    t0 = time.perf_counter()
    o = oracle.Oracle(g_np, cams[:1], tile_mask=mask)
    o.backward(d)
    dt = time.perf_counter() - t0
    oracle.set_threads(1)
    f = nt / T
    cores, model = host_cpu()
    sample = (f"view 0 of the {len(cams)}-view batch, {nt}/{T} of its 16x16 tiles, all "
              f"{g_np['means'].shape[0]} Gaussians projected, S1-S9, the C oracle on {threads} OpenMP threads "
              f"({cores} logical cores, {model}); value = sampled views / {dt:.2f} s")
    return f / dt, dt, sample


def cpu_baseline(cfg, g_np, cams, dL):
    th = oracle_threads()
    vps, dt, sample = oracle_sample(g_np, cams, dL, 1.0, threads=th)
    return {"value": round(vps, 5), "unit": UNIT, "cores": th, "kind": "oracle", "sample": sample}


def workload_config(cfg, P, Vr, N, V_all=None):
    V_all = Vr * N if V_all is None else V_all
    per = f"{Vr} views/GPU" if V_all == Vr * N else f"{V_all} views over {N} GPUs"
    return {"workload": f"{cfg.name}: {P} Gaussians SH{cfg.sh_degree}, {per} at {cfg.W}x{cfg.H}",
            "views_per_step": V_all, "global_batch_views": V_all, "parallelism": f"views dp{N}"}


def run_reference(args):
    """The base contract's reference arm for this tier: the oracle, timed as it stands on the
    host's cores, each step one full view of the same workload as the cpu_baseline leg."""
    ws, rank, _ = dist_setup()
    if rank != 0:
        return
    cfg = synth.CONFIGS[args.config]
    g_np, cams = synth.make_scene(cfg)
    dL = synth.make_dLdC(cfg.V, cfg.H, cfg.W, cfg.seed)
    th = oracle_threads()
    for w in range(min(args.warmup, 1)):
        oracle_sample(g_np, cams, dL, 1.0, threads=th)
    vals, times = [], []
    for k in range(args.steps):
        vps, dt, sample = oracle_sample(g_np, cams, dL, 1.0, threads=th)
        vals.append(vps)
        times.append(dt)
    value = len(vals) / sum(1.0 / v for v in vals)  # total sampled views / total time
    N = args.gpus if ws == 1 else ws
    conf = workload_config(cfg, cfg.P, cfg.V, 1)
    conf["sample"] = sample
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 5), "unit": UNIT,
            "n_gpus": N, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1e3 * statistics.mean(times), 2), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (mvgs-synth v1, seeded)",
            "config": conf,
            "cpu_baseline": {"value": round(value, 5), "unit": UNIT, "cores": th, "kind": "oracle", "sample": sample},
            "e2e": {"value": round(value, 5), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: relaunch under torch.distributed.run (the driver's own launch line)
        import socket
        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
        sk.close()
        os.execv(sys.executable, [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                                  f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
                                  "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]])
    if args.impl == "reference":
        run_reference(args)
    else:
        run_mvgs(args)


if __name__ == "__main__":
    main()
