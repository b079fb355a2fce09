"""NEXT-3 parity: the multi-view ADC step through the C ABI (mvgs_adc_step / mvgs_adc_remap)
against oracle/adc.py.  Decisions, order, origins, kinds and the report are
integer work: bit-exact.  Copied parameters (kept rows, clones, quats / opacity / SH of children)
are bit-exact; children log-scales are one fp32 subtraction on both sides: bit-exact; children
means are fp32 on the GPU vs fp64 in the oracle: |Δ| ≤ 1e-6 + 2e-6·(|μ| + Σ|R s n|)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from oracle import adc as oadc

pytestmark = pytest.mark.gpu


def dev_dict(d):
    return {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in d.items() if isinstance(v, np.ndarray)}


def gpu_adc(g, acc, noise, cfg, capacity=None):
    from paper_2506_12727_b200 import mvgs
    P = g["means"].shape[0]
    N = cfg["split_count"]
    cap = capacity if capacity is not None else P * (N + 1) + 1
    ctx = mvgs.create(0)
    try:
        gd = dev_dict(g)
        gd["sh_degree"] = g["sh_degree"]
        ad = {k + "_acc" if k != "denom" else "denom_acc": v for k, v in dev_dict(acc).items()}
        out = mvgs.alloc_gaussians(cap, g["sh"].shape[1], "cuda")
        origin = torch.empty(cap, dtype=torch.int32, device="cuda")
        kind = torch.empty(cap, dtype=torch.uint8, device="cuda")
        rep = mvgs.adc_step(ctx, gd, ad, torch.from_numpy(noise).cuda(), cfg, out, origin, kind)
        n = rep["P_new"]
        res = {k: v[:n].cpu().numpy() for k, v in out.items()}
        res["origin"] = origin[:n].cpu().numpy()
        res["kind"] = kind[:n].cpu().numpy()
        return res, rep
    finally:
        mvgs.destroy(ctx)


def compare(res, rep, ref, ref_rep, g, noise):
    assert rep == ref_rep
    np.testing.assert_array_equal(res["origin"], ref["origin"])
    np.testing.assert_array_equal(res["kind"], ref["kind"])
    for k in ("log_scales", "quats", "opacity_logits", "sh"):
        np.testing.assert_array_equal(res[k], ref[k], err_msg=k)
    ch = ref["kind"] == oadc.SPLIT
    np.testing.assert_array_equal(res["means"][~ch], ref["means"][~ch].astype(np.float32))
    if ch.any():
        o = ref["origin"][ch]
        bound = np.abs(g["means"][o]) + np.exp(g["log_scales"][o].astype(np.float64)).max(1, keepdims=True) \
            * np.abs(noise[o]).sum((1, 2))[:, None]
        assert np.all(np.abs(res["means"][ch] - ref["means"][ch]) <= 1e-6 + 2e-6 * bound)


@pytest.mark.parametrize("mode,N,psm", [(1, 2, 0.0), (0, 2, 0.0), (1, 3, 0.05), (0, 4, 0.05)])
def test_adc_step_matches_oracle(require_gpu, mode, N, psm):
    g, acc, noise = synth.make_adc_inputs(20000 + 37, 5 + N, N=N)
    cfg = oadc.default_config(metric_mode=mode, split_count=N, batch_views=4, prune_scale_max=psm)
    res, rep = gpu_adc(g, acc, noise, cfg)
    ref, ref_rep = oadc.adc_step(g, acc, noise, cfg)
    assert ref_rep["n_split"] > 100 and ref_rep["n_clone"] > 100 and ref_rep["n_pruned"] > 100
    compare(res, rep, ref, ref_rep, g, noise)


def test_adc_step_capacity_error_writes_nothing(require_gpu):
    from paper_2506_12727_b200 import mvgs
    g, acc, noise = synth.make_adc_inputs(3000, 1)
    cfg = oadc.default_config(batch_views=4)
    _, ref_rep = oadc.adc_step(g, acc, noise, cfg)
    with pytest.raises(mvgs.MvgsError) as ei:
        gpu_adc(g, acc, noise, cfg, capacity=ref_rep["P_new"] - 1)
    assert ei.value.status == mvgs.MVGS_ERR_CAPACITY and ei.value.report == ref_rep
    res, rep = gpu_adc(g, acc, noise, cfg, capacity=ref_rep["P_new"])
    assert rep == ref_rep


def test_adc_step_degenerate_cases(require_gpu):
    g, acc, noise = synth.make_adc_inputs(1000, 2)
    # everything pruned: prune_opacity × B ≥ 1
    res, rep = gpu_adc(g, acc, noise, oadc.default_config(prune_opacity=0.3, batch_views=4))
    assert rep["P_new"] == 0 and rep["n_pruned"] == 1000 + rep["n_split"] + rep["n_clone"]
    # zero accumulators: nothing densified, prune only
    z = {k: np.zeros_like(v) for k, v in acc.items()}
    res, rep = gpu_adc(g, z, noise, oadc.default_config(batch_views=2))
    ref, ref_rep = oadc.adc_step(g, z, noise, oadc.default_config(batch_views=2))
    compare(res, rep, ref, ref_rep, g, noise)
    # P = 0
    e = {k: v[:0] for k, v in g.items() if isinstance(v, np.ndarray)}
    e["sh_degree"] = 3
    res, rep = gpu_adc(e, {k: v[:0] for k, v in acc.items()}, noise[:0], oadc.default_config())
    assert rep == dict(n_split=0, n_clone=0, n_pruned=0, P_new=0)


def test_adc_remap_matches_oracle(require_gpu):
    from paper_2506_12727_b200 import mvgs
    g, acc, noise = synth.make_adc_inputs(5000, 3)
    cfg = oadc.default_config(batch_views=4)
    res, rep = gpu_adc(g, acc, noise, cfg)
    state = np.random.default_rng(0).normal(size=(5000, 16, 3)).astype(np.float32)
    ctx = mvgs.create(0)
    try:
        dst = torch.empty((rep["P_new"], 16, 3), device="cuda")
        mvgs.adc_remap(ctx, torch.from_numpy(state).cuda(), dst, torch.from_numpy(res["origin"]).cuda(),
                       torch.from_numpy(res["kind"]).cuda(), rep["P_new"])
        np.testing.assert_array_equal(dst.cpu().numpy(), oadc.remap(state, res["origin"], res["kind"]))
    finally:
        mvgs.destroy(ctx)


def test_full_size_sampled(require_gpu):
    """3 M Gaussians (garden scale): count identity on the whole set and, for a sample of
    parents, rows identical to the oracle run on those parents alone."""
    P = 3_000_000
    g, acc, noise = synth.make_adc_inputs(P, 11)
    cfg = oadc.default_config(batch_views=4, prune_scale_max=0.1)
    res, rep = gpu_adc(g, acc, noise, cfg, capacity=int(P * 1.6))
    assert rep["P_new"] == P + rep["n_split"] + rep["n_clone"] - rep["n_pruned"]
    assert np.all(np.diff(res["origin"]) >= 0)
    idx = np.sort(np.random.default_rng(1).choice(P, 4000, replace=False))
    sub = lambda d: {k: (v[idx] if isinstance(v, np.ndarray) else v) for k, v in d.items()}
    ref, ref_rep = oadc.adc_step(sub(g), sub(acc), noise[idx], cfg)
    sel = np.isin(res["origin"], idx)
    got = {k: v[sel] for k, v in res.items()}
    got["origin"] = np.searchsorted(idx, got["origin"]).astype(np.int32)
    compare(got, dict(n_split=ref_rep["n_split"], n_clone=ref_rep["n_clone"], n_pruned=ref_rep["n_pruned"],
                      P_new=int(sel.sum())), ref, ref_rep, sub(g), noise[idx])


def test_accumulators_and_fig_gradient_scenario_on_gpu(require_gpu):
    """The *_acc outputs of mvgs_adc_stats accumulate (two identical steps → exactly 2×), and the
    Fig. "gradient" scenario end to end on the GPU: E_old ≈ 0 → no densification with
    the single-view metric; E1/E2 > 0 → split with the multi-view metric."""
    from paper_2506_12727_b200 import mvgs
    W = H = 32
    g = dict(means=np.array([[0.3, 0.1, 0.0]], np.float32), log_scales=np.full((1, 3), np.log(0.08), np.float32),
             quats=np.array([[1, 0, 0, 0]], np.float32), opacity_logits=np.array([np.log(4.0)], np.float32),
             sh=np.zeros((1, 16, 3), np.float32), sh_degree=3)
    cams = synth.cams_array([synth.make_camera(np.eye(3), [0, 0, 5], W, H, 40.0),
                             synth.make_camera(np.diag([-1.0, -1.0, 1.0]), [0, 0, 5], W, H, 40.0)])
    rng = np.random.default_rng(0)
    d1 = rng.uniform(-1, 1, (3, H, W)).astype(np.float32) + np.linspace(0, 1, W, dtype=np.float32)
    dL = torch.from_numpy(np.ascontiguousarray(np.stack([d1, d1[:, ::-1, ::-1]]))).cuda()
    R = mvgs.Rasterizer(0)
    gd = dev_dict(g)
    gd["sh_degree"] = 3
    acc = {k: torch.zeros(1, device="cuda") for k in ("e1_acc", "e2_acc", "e_old_acc", "denom_acc")}
    for _ in range(2):
        R.preprocess(gd, cams)
        rgb, Tf, nc = R.alloc_forward()
        mvgs.render_fwd(R.ctx, rgb, Tf, nc)
        mvgs.render_bwd(R.ctx, dL, Tf, nc)
        grads, a = R.alloc_backward()
        a.update(acc)
        mvgs.adc_stats(R.ctx, grads, a)
    torch.cuda.synchronize()
    for k in ("e1", "e2", "e_old"):
        assert float(acc[k + "_acc"]) == 2 * float(a[k])
    assert float(acc["denom_acc"]) == 4.0
    e2 = float(a["e2"])
    assert e2 > 0 and float(a["e_old"]) < 1e-3 * e2
    acc_np = dict(e1=acc["e1_acc"].cpu().numpy(), e2=acc["e2_acc"].cpu().numpy(),
                  e_old=acc["e_old_acc"].cpu().numpy(), denom=acc["denom_acc"].cpu().numpy())
    z = np.zeros((1, 2, 3), np.float32)
    thr = dict(grad_threshold_split=e2 / 4, grad_threshold_clone=e2 / 4, size_threshold=0.01)
    _, rep0 = gpu_adc(g, acc_np, z, oadc.default_config(metric_mode=0, **thr))
    _, rep1 = gpu_adc(g, acc_np, z, oadc.default_config(metric_mode=1, **thr))
    assert rep0["n_split"] + rep0["n_clone"] == 0 and rep1["n_split"] == 1
    del R
