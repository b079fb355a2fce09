"""Oracle for NEXT-3: the multi-view adaptive density control step (P:4).
TEST INFRASTRUCTURE ONLY (same import rules as oracle/__init__.py: only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline leg may use it).

What the step computes, in the paper's terms:
  "For every predefined interval, Gaussians with a larger mean than a predefined threshold are
   chosen, and ADC splits large Gaussians to have smaller sizes and clones small Gaussians" (P:4)
  "E1 is good at splitting, and E2 is good at cloning"
  "the threshold hyperparameter for pruning Gaussians was multiplied by the number of images"

Readings (R35–R42), followed step by step below:
  mean        Ē = E_acc / denom_acc in fp32 (denom = Σ over steps of the views the Gaussian was
              visible in, R21); denom 0 → Ē = 0.
  large       max_k log_scale_k > fp32(ln size_threshold)   (world-space size gate, 3DGS)
  split       Ē1 ≥ τ_split ∧ large        (metric_mode multi_view; e_old mode uses Ē_old)
  clone       Ē2 ≥ τ_clone ∧ ¬large       (metric_mode multi_view; e_old mode uses Ē_old)
  split child k < N: mean + R(q̂)·(exp(log_scale) ⊙ n_k), n_k the caller's standard normal
              (3DGS: samples from the parent's own density), log_scale − fp32(ln split_factor),
              quats / opacity / SH copied.
  clone       verbatim copy.
  prune       every emitted Gaussian (kept, clone, child) with opacity logit <
              fp32(logit(prune_opacity·B)) or, when prune_scale_max > 0, max log_scale >
              fp32(ln prune_scale_max).
  order       for g = 0..P−1: [g unless split], [its clone], [its N children], prune-compacted.
Decisions are taken in fp32 exactly as the kernel takes them (DESIGN.md §4 rule: where floating
point decides an integer both sides use the same precision); values (child means) in fp64.
"""
from __future__ import annotations

import numpy as np

KEEP, CLONE, SPLIT = 0, 1, 2


def default_config(**kw):
    cfg = dict(grad_threshold_split=2e-4, grad_threshold_clone=2e-4, size_threshold=0.01, split_factor=1.6,
               split_count=2, prune_opacity=0.005, prune_scale_max=0.0, metric_mode=1, batch_views=1)
    cfg.update(kw)
    return cfg


def _f32(x):
    return np.float32(x)


def thresholds(cfg):
    """Host-side thresholds, fp64 math rounded once to fp32 (both sides do this)."""
    f = np.float64
    p = f(_f32(cfg["prune_opacity"])) * cfg["batch_views"]
    if p >= 1.0:
        logit_thr = np.float32(np.inf)
    elif p <= 0.0:
        logit_thr = np.float32(-np.inf)
    else:
        logit_thr = _f32(np.log(p / (1.0 - p)))
    psm = f(_f32(cfg["prune_scale_max"]))
    return dict(ln_size=_f32(np.log(f(_f32(cfg["size_threshold"])))),
                ln_split=_f32(np.log(f(_f32(cfg["split_factor"])))),
                logit_prune=logit_thr,
                ln_prune_scale=_f32(np.log(psm)) if psm > 0 else np.float32(np.inf),
                tau_split=_f32(cfg["grad_threshold_split"]), tau_clone=_f32(cfg["grad_threshold_clone"]))


def rotation(q):
    """R(q̂) for q = (w, x, y, z), q̂ = q/‖q‖ (the standard unit-quaternion matrix)."""
    q = np.asarray(q, np.float64)
    w, x, y, z = q / np.linalg.norm(q)
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


def adc_step(g, acc, noise, cfg):
    """g: dict of float32 arrays (means [P,3], log_scales [P,3], quats [P,4], opacity_logits [P],
    sh [P,S,3]); acc: dict of float32 e1, e2, e_old, denom [P]; noise [P,N,3] float32.
    Returns (out dict of arrays incl. 'origin' int32 and 'kind' uint8, report dict)."""
    th = thresholds(cfg)
    N = int(cfg["split_count"])
    P = g["means"].shape[0]
    den = np.asarray(acc["denom"], np.float32)

    def mean(e):
        e = np.asarray(e, np.float32)
        with np.errstate(divide="ignore", invalid="ignore"):
            m = (e / np.where(den > 0, den, np.float32(1))).astype(np.float32)
        return np.where(den > 0, m, np.float32(0))

    ls = np.asarray(g["log_scales"], np.float32)
    large = ls.max(1) > th["ln_size"]
    if cfg["metric_mode"] == 1:
        m_split, m_clone = mean(acc["e1"]), mean(acc["e2"])
    else:
        m_split = m_clone = mean(acc["e_old"])
    split = (m_split >= th["tau_split"]) & large
    clone = (m_clone >= th["tau_clone"]) & ~large
    ol = np.asarray(g["opacity_logits"], np.float32)

    rows = []  # (origin, kind, mean, log_scale)
    n_pruned = 0
    for i in range(P):
        items = []
        if not split[i]:
            items.append((KEEP, g["means"][i].astype(np.float64), ls[i]))
        if clone[i]:
            items.append((CLONE, g["means"][i].astype(np.float64), ls[i]))
        if split[i]:
            R = rotation(g["quats"][i])
            s = np.exp(ls[i].astype(np.float64))
            child_ls = (ls[i] - th["ln_split"]).astype(np.float32)
            for k in range(N):
                m = g["means"][i].astype(np.float64) + R @ (s * noise[i, k].astype(np.float64))
                items.append((SPLIT, m, child_ls))
        for kind, m, l in items:
            if ol[i] < th["logit_prune"] or l.max() > th["ln_prune_scale"]:
                n_pruned += 1
                continue
            rows.append((i, kind, m, l))
    n = len(rows)
    origin = np.array([r[0] for r in rows], np.int32).reshape(n)
    out = dict(origin=origin, kind=np.array([r[1] for r in rows], np.uint8).reshape(n),
               means=np.array([r[2] for r in rows], np.float64).reshape(n, 3),
               log_scales=np.array([r[3] for r in rows], np.float32).reshape(n, 3),
               quats=g["quats"][origin], opacity_logits=g["opacity_logits"][origin], sh=g["sh"][origin])
    report = dict(n_split=int(split.sum()), n_clone=int(clone.sum()), n_pruned=n_pruned, P_new=n)
    return out, report


def remap(src, origin, kind):
    """Optimizer-state resize: kept Gaussians keep their row, clones and split children start at 0."""
    src = np.asarray(src)
    out = src[origin].copy()
    out[kind != KEEP] = 0
    return out
