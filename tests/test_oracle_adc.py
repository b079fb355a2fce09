"""Pins for the NEXT-3 oracle (oracle/adc.py): the multi-view ADC step (P:4).
Each pin checks the oracle against something other than itself: SPEC's worked examples
(S:374–376), the count identity, textbook Gaussian sampling (child means of a split are
draws from the parent's N(μ, RS²Rᵀ)), a closed-form rotation, and the Fig. "gradient" scenario
run through the oracle rasterizer (two views whose 2D gradients cancel)."""
import numpy as np

import oracle
import synth
from oracle import adc


def one_gaussian(log_scale, opacity=0.9, q=(1, 0, 0, 0), mean=(0, 0, 0)):
    return dict(means=np.array([mean], np.float32), log_scales=np.array([log_scale], np.float32),
                quats=np.array([q], np.float32),
                opacity_logits=np.array([np.log(opacity / (1 - opacity))], np.float32),
                sh=np.arange(48, dtype=np.float32).reshape(1, 16, 3), sh_degree=3)


def acc_of(e1, e2, eo, den):
    f = lambda v: np.atleast_1d(np.asarray(v, np.float32))
    return dict(e1=f(e1), e2=f(e2), e_old=f(eo), denom=f(den))


def test_zero_accumulators_no_densify_but_prune_applies():
    """all accumulators zero → no split, no clone; prune still applies."""
    g, acc, noise = synth.make_adc_inputs(500, 1)
    z = {k: np.zeros_like(v) for k, v in acc.items()}
    cfg = adc.default_config(batch_views=4)
    out, rep = adc.adc_step(g, z, noise, cfg)
    o = 1 / (1 + np.exp(-g["opacity_logits"].astype(np.float64)))
    assert np.min(np.abs(o - 0.02)) > 1e-6  # no Gaussian within rounding of the threshold
    assert rep["n_split"] == 0 and rep["n_clone"] == 0 and rep["n_pruned"] == int(np.sum(o < 0.02)) > 0
    np.testing.assert_array_equal(out["origin"], np.nonzero(o >= 0.02)[0])
    assert np.all(out["kind"] == adc.KEEP)


def test_clone_semantics_single_gaussian():
    """one Gaussian, E_old mean = 2·threshold, tiny scale → cloned, count 1 → 2, identical."""
    g = one_gaussian([np.log(1e-3)] * 3)
    for mode in (0, 1):
        cfg = adc.default_config(metric_mode=mode)
        out, rep = adc.adc_step(g, acc_of(4e-4, 4e-4, 4e-4, 1), np.zeros((1, 2, 3), np.float32), cfg)
        assert rep == dict(n_split=0, n_clone=1, n_pruned=0, P_new=2)
        assert list(out["kind"]) == [adc.KEEP, adc.CLONE]
        for k in ("means", "log_scales", "quats", "opacity_logits", "sh"):
            np.testing.assert_array_equal(out[k][0], out[k][1])
            np.testing.assert_array_equal(np.asarray(out[k][0], np.float64), np.asarray(g[k][0], np.float64))


def test_count_identity_and_disjoint_sets():
    """P_new = P + (N−1)·|split| + |clone| − |pruned|; split and clone are disjoint."""
    for N in (2, 3):
        g, acc, noise = synth.make_adc_inputs(3000, 2, N=N)
        cfg = adc.default_config(split_count=N, batch_views=4, prune_scale_max=0.2)
        out, rep = adc.adc_step(g, acc, noise, cfg)
        P = 3000
        assert rep["P_new"] == P + (N - 1) * rep["n_split"] + rep["n_clone"] - rep["n_pruned"]
        assert len(out["origin"]) == rep["P_new"]
        assert rep["n_split"] > 50 and rep["n_clone"] > 50 and rep["n_pruned"] > 50
        # no origin is both split (kind 2) and kept or cloned
        s = set(out["origin"][out["kind"] == adc.SPLIT])
        assert not s & set(out["origin"][out["kind"] != adc.SPLIT])
        assert np.all(np.diff(out["origin"]) >= 0)  # canonical order


def test_split_children_sample_parent_density():
    """Children means are μ + R(q̂)(s ⊙ n): with n ~ N(0, I) their covariance is R S² Rᵀ
    (textbook); anisotropic scales and a generic rotation catch a transposed R or swapped axes."""
    rng = np.random.default_rng(3)
    n = 40000
    q = np.array([0.8, 0.3, -0.4, 0.35])
    ls = np.log([0.3, 0.1, 0.02])
    g = one_gaussian(ls, q=q, mean=(1.0, -2.0, 0.5))
    g = {k: (np.repeat(v, n, 0) if isinstance(v, np.ndarray) else v) for k, v in g.items()}
    noise = rng.normal(0, 1, (n, 2, 3)).astype(np.float32)
    out, rep = adc.adc_step(g, acc_of([1.0] * n, [1.0] * n, [1.0] * n, [1.0] * n), noise,
                            adc.default_config(size_threshold=0.05))
    assert rep["n_split"] == n and rep["P_new"] == 2 * n
    m = out["means"]
    w, x, y, z = q / np.linalg.norm(q)
    # closed form of R(q̂) written independently, column by column (image of the basis vectors)
    ex = [w * w + x * x - y * y - z * z, 2 * (x * y + w * z), 2 * (x * z - w * y)]
    ey = [2 * (x * y - w * z), w * w - x * x + y * y - z * z, 2 * (y * z + w * x)]
    ez = [2 * (x * z + w * y), 2 * (y * z - w * x), w * w - x * x - y * y + z * z]
    R = np.array([ex, ey, ez]).T
    S2 = np.diag(np.exp(2 * ls))
    cov = np.cov((m - [1.0, -2.0, 0.5]).T)
    np.testing.assert_allclose(cov, R @ S2 @ R.T, atol=0.03 * 0.09)
    np.testing.assert_allclose(m.mean(0), [1.0, -2.0, 0.5], atol=4 * 0.3 / np.sqrt(2 * n))
    # child scale = parent / split_factor (fp32 log-domain subtraction)
    np.testing.assert_allclose(np.exp(out["log_scales"][0].astype(np.float64)), np.exp(ls) / 1.6, rtol=1e-6)


def test_rotation_closed_form():
    th = 0.7
    R = adc.rotation([np.cos(th / 2), 0, 0, np.sin(th / 2)])
    np.testing.assert_allclose(R @ [1, 0, 0], [np.cos(th), np.sin(th), 0], atol=1e-15)
    R = adc.rotation([0.2, -0.5, 0.7, 0.1])
    np.testing.assert_allclose(R @ R.T, np.eye(3), atol=1e-14)
    assert abs(np.linalg.det(R) - 1) < 1e-14


def test_prune_threshold_scales_with_batch_views():
    """pruning threshold × number of images — opacity 0.01 survives B = 1, pruned at B = 4."""
    g = one_gaussian([np.log(1e-3)] * 3, opacity=0.01)
    a = acc_of(0, 0, 0, 0)
    z = np.zeros((1, 2, 3), np.float32)
    assert adc.adc_step(g, a, z, adc.default_config(batch_views=1))[1]["P_new"] == 1
    assert adc.adc_step(g, a, z, adc.default_config(batch_views=4))[1]["P_new"] == 0


def test_remap_zeroes_new_rows():
    origin = np.array([0, 0, 2, 2, 3], np.int32)
    kind = np.array([0, 1, 2, 2, 0], np.uint8)
    src = np.arange(8, dtype=np.float32).reshape(4, 2)
    np.testing.assert_array_equal(adc.remap(src, origin, kind), [[0, 1], [0, 0], [0, 0], [0, 0], [6, 7]])


def test_fig_gradient_scenario_through_the_rasterizer():
    """P:4–9 / S:376: two views whose per-view 2D positional gradients cancel (the second camera
    is the first rolled by 180° about its axis and sees the mirrored ∂L/∂C) → E_old ≈ 0 while
    E1, E2 > 0; ADC with E_old does not densify, multi-view ADC does."""
    W = H = 32
    g = one_gaussian([np.log(0.08)] * 3, opacity=0.8, mean=(0.3, 0.1, 0.0))
    g["sh"][:] = 0
    cams = synth.cams_array([synth.make_camera(np.eye(3), [0, 0, 5], W, H, 40.0),
                             synth.make_camera(np.diag([-1.0, -1.0, 1.0]), [0, 0, 5], W, H, 40.0)])
    rng = np.random.default_rng(0)
    d1 = rng.uniform(-1, 1, (3, H, W)).astype(np.float32) + np.linspace(0, 1, W, dtype=np.float32)
    dL = np.stack([d1, d1[:, ::-1, ::-1]])
    o = oracle.Oracle(g, cams)
    o.forward()
    r = o.backward(np.ascontiguousarray(dL))
    e1, e2, eo = float(r["e1"][0]), float(r["e2"][0]), float(r["e_old"][0])
    assert e1 >= e2 > 1e3 * max(eo, 1e-30) and e2 > 0
    thr = 0.5 * e2 / 2
    acc = acc_of(e1, e2, eo, 2)
    z = np.zeros((1, 2, 3), np.float32)
    cfg = dict(grad_threshold_split=thr, grad_threshold_clone=thr, size_threshold=0.01)
    _, rep_old = adc.adc_step(g, acc, z, adc.default_config(metric_mode=0, **cfg))
    _, rep_mv = adc.adc_step(g, acc, z, adc.default_config(metric_mode=1, **cfg))
    assert rep_old["n_split"] + rep_old["n_clone"] == 0
    assert rep_mv["n_split"] == 1  # large (0.08 > 0.01): E1 splits it


def test_single_view_e2_equals_e_old_and_clone_sets_agree():
    """with one view E2 = E_old, so multi-view clone set = E_old clone set."""
    cfg_s = synth.scaled(synth.CONFIGS["tiny"], P=300, V=1, W=48, H=40)
    g, cams = synth.make_scene(cfg_s)
    o = oracle.Oracle(g, cams)
    o.forward()
    r = o.backward(synth.make_dLdC_scaled(1, 40, 48, 3))
    np.testing.assert_allclose(r["e2"], r["e_old"], rtol=1e-6, atol=0)
    acc = acc_of(r["e1"], r["e2"], r["e_old"], r["vis"])
    tau = float(np.median(r["e2"][r["vis"] > 0]))
    z = np.zeros((300, 2, 3), np.float32)
    kw = dict(grad_threshold_clone=tau, grad_threshold_split=1e9, size_threshold=0.08)
    a, ra = adc.adc_step(g, acc, z, adc.default_config(metric_mode=0, **kw))
    b, rb = adc.adc_step(g, acc, z, adc.default_config(metric_mode=1, **kw))
    assert ra["n_clone"] > 10
    np.testing.assert_array_equal(a["origin"][a["kind"] == 1], b["origin"][b["kind"] == 1])
