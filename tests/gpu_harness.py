"""Shared helpers for the GPU parity tests: run the CUDA path through the C ABI
on synth inputs and compare with the oracle under the DESIGN.md §5 rules."""
import numpy as np
import torch


def to_dev(g, device="cuda"):
    out = {k: torch.from_numpy(np.ascontiguousarray(v)).to(device) for k, v in g.items() if isinstance(v, np.ndarray)}
    out["sh_degree"] = g["sh_degree"]
    return out


def run_gpu(g, cams, dLdC=None, bg=(0.0, 0.0, 0.0), max_pairs=0, max_entries=0, export=True):
    from paper_2506_12727_b200 import mvgs
    R = mvgs.Rasterizer(0, max_pairs, max_entries)
    gd = to_dev(g)
    R.preprocess(gd, cams, bg)
    rgb, Tf, nc = R.forward()
    out = dict(stats=R.stats)
    if dLdC is not None:
        nbl = None
        if export:  # the backward's own blended-entry count per pixel (its re-taken decisions)
            nbl = torch.full((len(cams), R.H, R.W), -1, dtype=torch.int32, device="cuda")
            mvgs.set_debug_blend_counts(R.ctx, nbl)
        grads, adc = R.backward(torch.from_numpy(np.ascontiguousarray(dLdC, np.float32)).cuda())
        if nbl is not None:
            mvgs.set_debug_blend_counts(R.ctx, None)
            out["bwd_nblend"] = nbl.cpu().numpy()
        out.update({k: v.cpu().numpy() for k, v in grads.items()})
        out.update({k: v.cpu().numpy() for k, v in adc.items()})
    torch.cuda.synchronize()
    out.update(rgb=rgb.cpu().numpy(), T_final=Tf.cpu().numpy(), n_contrib=nc.cpu().numpy())
    if export:
        st = R.stats
        V, T = len(cams), st["tiles_x"] * st["tiles_y"]
        Q, K = int(st["Q"]), int(st["K"])
        rs = torch.empty(V * T + 1, dtype=torch.int64, device="cuda")
        eg = torch.empty(max(K, 1), dtype=torch.int32, device="cuda")
        mvgs.export_lists(R.ctx, rs, eg)
        pid = torch.empty((max(Q, 1), 2), dtype=torch.int32, device="cuda")
        pi = torch.empty((max(Q, 1), 8), dtype=torch.int32, device="cuda")
        pf = torch.empty((max(Q, 1), 12), dtype=torch.float32, device="cuda")
        pg = torch.empty((max(Q, 1), 10), dtype=torch.float32, device="cuda")
        mvgs.export_pairs(R.ctx, pid, pi, pf, pg if dLdC is not None else None)
        torch.cuda.synchronize()
        out.update(range_start=rs.cpu().numpy(), entry_gid=eg.cpu().numpy()[:K], pair_ids=pid.cpu().numpy()[:Q],
                   pair_i=pi.cpu().numpy()[:Q], pair_f=pf.cpu().numpy()[:Q],
                   pair_g=pg.cpu().numpy()[:Q] if dLdC is not None else None)
    del R
    return out


def assert_close_rel(got, ref, name, rtol=1e-3, floor=1e-6, scale=None, ctol=1e-4, sens=None, max_sens_frac=1e-3):
    """per tensor ‖Δ‖/‖ref‖ ≤ rtol and per element
    |Δ| ≤ rtol·|ref| + ctol·(scale + ‖scale row‖) + floor·max|ref|, where `scale`
    (optional, default |ref|) is the magnitude of the per-view terms the element sums
    (Σ_v |ref_v|): an element that is a cancellation of larger per-view terms is held to
    fp32 accuracy of those terms, not of the cancelled result; and a component of a
    Gaussian's gradient row (its 3 mean components, 4 quaternion components, SH
    coefficients …, axis 0 = Gaussian) is held to that accuracy relative to the row's
    norm, since the chain rule mixes the row's components through rotations and
    Jacobians (a component that cancels to ~1e-5 of its row carries the row's rounding).
    `sens` (optional): the oracle's own change under a 1-ulp perturbation of its fp32 inputs
    (input_sensitivity); an element may also deviate by 2·sens — it is ill-conditioned at the
    fp32 input level, so no fp32 implementation resolves it better — but at most
    max_sens_frac of the elements may need that allowance.  Reports the worst elements."""
    g0 = np.asarray(got, np.float64)
    r0 = np.asarray(ref, np.float64)
    s0 = np.abs(r0) if scale is None else np.asarray(scale, np.float64)
    if r0.ndim >= 2 and r0.shape[0] > 0:
        rown = np.linalg.norm(s0.reshape(r0.shape[0], -1), axis=1)
        rown = np.broadcast_to(rown.reshape((-1,) + (1,) * (r0.ndim - 1)), r0.shape).reshape(-1)
    else:
        rown = np.zeros(r0.size)
    got = g0.reshape(-1)
    ref = r0.reshape(-1)
    sc = (np.zeros_like(ref) if scale is None else s0.reshape(-1)) + rown
    assert got.shape == ref.shape, name
    d = np.abs(got - ref)
    nref = np.linalg.norm(ref)
    mx = np.max(np.abs(ref)) if ref.size else 0.0
    if nref == 0:
        assert np.all(d <= 1e-30 + 1e-12), name
        return
    rel = np.linalg.norm(got - ref) / nref
    lim = rtol * np.abs(ref) + ctol * sc + floor * mx
    if sens is not None:
        sv = 2.0 * np.asarray(sens, np.float64).reshape(-1)
        need = (d > lim) & (d <= sv)
        assert need.mean() <= max_sens_frac, f"{name}: {need.sum()} elements need the input-sensitivity allowance"
        lim = np.maximum(lim, sv)
    bad = np.argsort(-(d - lim))[:10]
    msg = f"{name}: tensor rel {rel:.3e}; worst " + ", ".join(
        f"[{i}] got {got[i]:.6e} ref {ref[i]:.6e} lim {lim[i]:.3e}" for i in bad[:5])
    assert rel <= rtol, msg
    assert np.all(d <= lim), msg


def per_view_scale(g, cams, dLdC, bg=(0.0, 0.0, 0.0), tile_mask=None, extra=True):
    """Σ_v |gradient of view v alone| for every output (the oracle, one view at a time)."""
    import oracle
    out = None
    for v in range(len(cams)):
        m = None if tile_mask is None else tile_mask[v:v + 1]
        ov = oracle.Oracle(g, cams[v:v + 1], bg=bg, tile_mask=m)
        r = ov.backward(dLdC[v:v + 1])
        if extra:  # per-pair arrays: oracle-sized scenes only
            r["gsum"] = ov.adc_extra()["gsum"]
        if out is None:
            out = {k: np.abs(x) for k, x in r.items()}
        else:
            for k in out:
                out[k] = out[k] + np.abs(r[k])
    out["e_old"] = out["e2"]  # |Σ_v g_v| is a cancellation of terms of total size Σ_v |g_v| = E2
    return out


def input_sensitivity(g, cams, dLdC, keys, tile_mask=None, draws=3, bg=(0.0, 0.0, 0.0)):
    """max over `draws` seeded perturbations of |oracle(g', ∂L/∂C') − oracle(g, ∂L/∂C)| for
    `keys`: the fp32 means, log-scales, quaternions and every pixel's ∂L/∂C each moved by one
    ulp (random sign) — the part of a gradient that fp32 inputs, and fp32 rounding of the
    per-pixel terms it sums, cannot determine."""
    import oracle
    base = oracle.Oracle(g, cams, bg=bg, tile_mask=tile_mask).backward(dLdC)
    out = {k: np.zeros_like(base[k]) for k in keys}
    for t in range(draws):
        r = np.random.default_rng(1000 + t)
        g2 = dict(g)
        for k in ("means", "log_scales", "quats"):
            x = np.asarray(g[k], np.float32)
            g2[k] = (x * (1 + r.choice([-1.0, 1.0], x.shape) * 2.0 ** -23)).astype(np.float32)
        d2 = (np.asarray(dLdC, np.float32) * (1 + r.choice([-1.0, 1.0], np.shape(dLdC)) * 2.0 ** -23)).astype(np.float32)
        o = oracle.Oracle(g2, cams, bg=bg, tile_mask=tile_mask).backward(d2)
        for k in keys:
            out[k] = np.maximum(out[k], np.abs(o[k] - base[k]))
    return out
