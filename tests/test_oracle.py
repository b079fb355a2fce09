"""Pins for the CPU oracle (SURVEY.md §8(c) P1–P17), run with -m "not gpu".

Each test pins the oracle to something other than itself: a closed form, a
worked example printed in the paper (tests/golden/), finite differences, an
invariant, or brute force.  Citations are PAPER.md lines (P:n) and SPEC.md
lines (S:n).
"""
import math
import os

import numpy as np
import pytest

import oracle
import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
C0 = 0.28209479177387814


def scene(means, log_scales=None, quats=None, logits=None, sh=None, sh_degree=0):
    means = np.asarray(means, np.float32).reshape(-1, 3)
    P = len(means)
    K = (sh_degree + 1) ** 2
    return dict(
        means=means,
        log_scales=np.asarray(log_scales if log_scales is not None else np.full((P, 3), -3.0), np.float32).reshape(P, 3),
        quats=np.asarray(quats if quats is not None else np.tile([1, 0, 0, 0], (P, 1)), np.float32).reshape(P, 4),
        opacity_logits=np.asarray(logits if logits is not None else np.zeros(P), np.float32).reshape(P),
        sh=np.asarray(sh if sh is not None else np.zeros((P, K, 3)), np.float32).reshape(P, K, 3),
        sh_degree=sh_degree,
    )


def cam_identity(W=32, H=32, f=40.0, R=np.eye(3), t=(0, 0, 0), cx=None, cy=None):
    return synth.cams_array([synth.make_camera(R, t, W, H, f, cx=cx, cy=cy)])


# --------------------------------------------------------------------- CA exp
def test_ca_exp_is_an_exp():
    """§4.3 canonical exp: within 3 ulp of the true exp on its range, 0 below −87."""
    xs = np.concatenate([np.linspace(-87, 88, 20001), -np.logspace(-8, 1.9, 2000), [0.0]]).astype(np.float32)
    got = np.array([oracle.ca_exp(x) for x in xs], np.float64)
    ref = np.exp(xs.astype(np.float64))
    ulp = np.spacing(ref.astype(np.float32)).astype(np.float64)
    assert np.all(np.abs(got - ref) <= 3 * ulp) and np.mean(np.abs(got - ref) <= ulp) > 0.9
    assert oracle.ca_exp(-87.5) == 0.0 and oracle.ca_exp(0.0) == 1.0


# ----------------------------------------------------------- P1/P3 projection
def test_P3_isotropic_on_axis_conic_and_radius():
    """Isotropic s at depth z on the optical axis, fx=fy=f: Σ' = ((f s/z)² + 0.3) I,
    conic = I/σ'², radius = ⌈3√(σ'² + √0.1)⌉ (R5, R7)."""
    s, z, f = 0.05, 2.0, 40.0
    g = scene([0, 0, z], log_scales=np.full(3, math.log(s)))
    o = oracle.Oracle(g, cam_identity(f=f))
    p = o.pairs()
    s32 = float(np.exp(np.float32(math.log(s))))
    sig2 = (f * s32 / z) ** 2 + 0.3
    assert p["vis"][0, 0] == 1 and p["zvis"][0, 0] == 1
    np.testing.assert_allclose([p["A"][0, 0], p["B"][0, 0], p["C"][0, 0]], [1 / sig2, 0, 1 / sig2], rtol=2e-6, atol=1e-7)
    assert p["radius"][0, 0] == math.ceil(3 * math.sqrt(sig2 + math.sqrt(0.1)))
    # P2: on-axis ⇒ μ' = (cx, cy); depth = z
    assert p["px"][0, 0] == np.float32(15.5) and p["py"][0, 0] == np.float32(15.5)
    assert p["depth"][0, 0] == np.float32(z)


def test_P1_axis_swap_through_projection():
    """90° rotation about z swaps the x/y scales: Σ = R diag(a²,b²,c²) Rᵀ = diag(b²,a²,c²)
    (S:115), seen on-axis as conic = diag(1/((f b/z)²+0.3), 1/((f a/z)²+0.3))."""
    a, b, c, z, f = 0.08, 0.03, 0.05, 3.0, 50.0
    q = [math.cos(math.pi / 4), 0, 0, math.sin(math.pi / 4)]
    g = scene([0, 0, z], log_scales=[math.log(a), math.log(b), math.log(c)], quats=q)
    p = oracle.Oracle(g, cam_identity(f=f)).pairs()
    ea, eb = [float(np.exp(np.float32(math.log(v)))) for v in (a, b)]
    sx = (f * eb / z) ** 2 + 0.3
    sy = (f * ea / z) ** 2 + 0.3
    np.testing.assert_allclose([p["A"][0, 0], p["C"][0, 0]], [1 / sx, 1 / sy], rtol=1e-5)
    assert abs(p["B"][0, 0]) < 1e-6 * p["A"][0, 0]


def test_P2_b2_cameras_see_origin_at_centre():
    """Appendix B.2 pair (tests/golden/b2_cameras.txt, reading R23): both cameras see
    the origin at the image centre at depth 1."""
    rows = [l.split("|") for l in open(os.path.join(GOLDEN, "b2_cameras.txt")) if l.strip() and not l.startswith("#")]
    cams = synth.cams_array([synth.make_camera(np.array(r[1].split(), float).reshape(3, 3),
                                               np.array(r[2].split(), float), 33, 33, 30.0) for r in rows])
    p = oracle.Oracle(scene([0, 0, 0]), cams).pairs()
    for v, r in enumerate(rows):
        assert p["depth"][v, 0] == np.float32(float(r[3]))
        assert p["px"][v, 0] == np.float32(16.0) and p["py"][v, 0] == np.float32(16.0)


# -------------------------------------------------------------- P4/P5 blending
def test_P4_single_isotropic_footprint_and_alpha():
    """One isotropic Gaussian on the axis: n_contrib = 1 exactly on lattice pixels with
    ‖p − μ'‖² ≤ 2σ'² ln(255 o) inside its rect (α ≥ 1/255, R12), colour =
    rgb·α + (1−α)·bg with α = o·exp(−‖p−μ'‖²/2σ'²), T_final = 1 − α; elsewhere 0, bg, 1."""
    s, z, f, W = 0.06, 2.0, 40.0, 32
    logit = 0.3
    rgb = np.array([0.9, 0.4, 0.2])
    g = scene([0, 0, z], log_scales=np.full(3, math.log(s)), logits=[logit],
              sh=((rgb - 0.5) / C0).reshape(1, 1, 3))
    bg = np.array([0.1, 0.2, 0.3], np.float32)
    o = oracle.Oracle(g, cam_identity(W=W, H=W, f=f), bg=bg)
    im = o.forward()
    p = o.pairs()
    s64 = math.exp(float(np.float32(math.log(s))))  # fp64 value chain of the float input
    sig2 = (f * s64 / z) ** 2 + 0.3
    op = 1 / (1 + math.exp(-float(np.float32(logit))))
    thr = 2 * sig2 * math.log(255 * op)
    yy, xx = np.mgrid[0:W, 0:W]
    d2 = (xx - 15.5) ** 2 + (yy - 15.5) ** 2
    assert np.min(np.abs(d2 - thr)) > 1e-3 * thr  # parameters keep every pixel off the threshold
    inrect = ((xx // 16 >= p["rx0"][0, 0]) & (xx // 16 < p["rx1"][0, 0])
              & (yy // 16 >= p["ry0"][0, 0]) & (yy // 16 < p["ry1"][0, 0]))
    foot = (d2 <= thr) & inrect
    assert foot.sum() > 20 and (~foot).sum() > 20
    np.testing.assert_array_equal(im["n_contrib"][0], foot.astype(np.int32))
    alpha = np.where(foot, op * np.exp(-d2 / (2 * sig2)), 0.0)
    rgb32 = C0 * ((rgb - 0.5) / C0).astype(np.float32).astype(np.float64) + 0.5
    for ch in range(3):
        np.testing.assert_allclose(im["rgb"][0, ch], rgb32[ch] * alpha + (1 - alpha) * float(bg[ch]), atol=1e-12)
    np.testing.assert_allclose(im["T_final"][0], 1 - alpha, atol=1e-12)


def test_P5_two_cocentred_terms():
    """Front o₁=0.5 (c₁), back o₂=0.9 (c₂), both centred on a pixel: C = 0.5c₁ + 0.45c₂,
    T_final = 0.05 (Eq. 1; S:195 with o₂ reachable by a sigmoid, R13)."""
    c1, c2 = np.array([1.0, 0.0, 0.25]), np.array([0.0, 1.0, 0.5])
    g = scene([[0, 0, 2.0], [0, 0, 3.0]], log_scales=np.full((2, 3), math.log(0.05)),
              logits=[0.0, math.log(9.0)], sh=np.stack([(c1 - 0.5) / C0, (c2 - 0.5) / C0]).reshape(2, 1, 3))
    o = oracle.Oracle(g, cam_identity(W=33, H=33, f=40.0))
    im = o.forward()
    np.testing.assert_allclose(im["rgb"][0, :, 16, 16], 0.5 * c1 + 0.45 * c2, atol=1e-6)
    assert abs(im["T_final"][0, 16, 16] - 0.05) < 1e-6
    assert im["n_contrib"][0, 16, 16] == 2


def test_P8_early_termination_is_sound():
    """Disabling early termination changes no pixel by more than 2e-3."""
    g, cams = synth.make_scene("tiny")
    a = oracle.Oracle(g, cams).forward()
    b = oracle.Oracle(g, cams, flags=oracle.NO_EARLY_TERMINATION).forward()
    assert np.max(np.abs(a["rgb"] - b["rgb"])) <= 2e-3
    assert np.all(b["n_contrib"] >= a["n_contrib"])
    assert np.any(b["n_contrib"] > a["n_contrib"])  # termination actually happened


# --------------------------------------------------------------- P6/P7 lists
def test_P6_P7_lists_equal_brute_force():
    """Per-(view,tile) lists = brute-force O(Q·T) rect test sorted by the tuple
    (depth bits, gid) (R9/R10); rect = [3DGS] getRect re-derived in numpy."""
    g, cams = synth.make_scene(synth.scaled(synth.CONFIGS["tiny"], P=300))
    o = oracle.Oracle(g, cams)
    p = o.pairs()
    off, gid = o.lists()
    TX, TY = o.TX, o.TY
    # independent rect from (px, py, radius) in float32
    px, py, r = p["px"], p["py"], p["radius"].astype(np.float32)
    with np.errstate(invalid="ignore"):
        def lo(v, T):
            return np.where(~(v > 0), 0, np.where(v >= T, T, np.trunc(v))).astype(np.int64)
        rx0 = lo((px - r) * np.float32(0.0625), TX)
        ry0 = lo((py - r) * np.float32(0.0625), TY)
        rx1 = lo(((px + r) + np.float32(15)) * np.float32(0.0625), TX)
        ry1 = lo(((py + r) + np.float32(15)) * np.float32(0.0625), TY)
    vis = p["vis"].astype(bool)
    np.testing.assert_array_equal(rx0[vis], p["rx0"][vis])
    np.testing.assert_array_equal(rx1[vis], p["rx1"][vis])
    np.testing.assert_array_equal(ry0[vis], p["ry0"][vis])
    np.testing.assert_array_equal(ry1[vis], p["ry1"][vis])
    for v in range(o.V):
        for t in range(o.T):
            tx, ty = t % TX, t // TX
            members = [i for i in range(o.P) if vis[v, i] and rx0[v, i] <= tx < rx1[v, i] and ry0[v, i] <= ty < ry1[v, i]]
            members.sort(key=lambda i: (int(p["depth"][v, i].view(np.uint32)), i))
            b = v * o.T + t
            assert list(gid[off[b]:off[b + 1]]) == members


# -------------------------------------------------------------- gradients
def _loss(g, cams, dLdC, bg=(0, 0, 0)):
    o = oracle.Oracle(g, cams, bg=bg)
    im = o.forward()
    return float(np.sum(im["rgb"] * dLdC)), im["n_contrib"], (o.lists()[1], o.decision_hash())


def _fd_check(g, cams, dLdC, bg=(0.0, 0.0, 0.0), h=1e-3, rtol=1e-4, atol=1e-7, keys=None):
    """Central differences with one Richardson step (error O(h⁴)) on the float32 inputs;
    the actual representable step is used as the divisor."""
    o = oracle.Oracle(g, cams, bg=bg)
    grads = o.backward(dLdC)
    _, nc0, l0 = _loss(g, cams, dLdC, bg)
    gk = {"means": "d_means", "log_scales": "d_log_scales", "quats": "d_quats",
          "opacity_logits": "d_opacity_logits", "sh": "d_sh"}
    checked = 0

    def central(key, idx, step):
        gp = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in g.items()}
        gm = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in g.items()}
        base = g[key].reshape(-1)[idx]
        gp[key].reshape(-1)[idx] = base + np.float32(step)
        gm[key].reshape(-1)[idx] = base - np.float32(step)
        delta = float(gp[key].reshape(-1)[idx]) - float(gm[key].reshape(-1)[idx])
        lp, ncp, lsp = _loss(gp, cams, dLdC, bg)
        lm, ncm, lsm = _loss(gm, cams, dLdC, bg)
        smooth = (np.array_equal(ncp, nc0) and np.array_equal(ncm, nc0)
                  and np.array_equal(lsp[0], l0[0]) and np.array_equal(lsm[0], l0[0])
                  and lsp[1] == l0[1] and lsm[1] == l0[1])
        return (lp - lm) / delta, smooth

    for key, gname in gk.items():
        if keys and key not in keys:
            continue
        arr = g[key]
        ana = grads[gname].reshape(-1)
        for idx in range(arr.size):
            if key == "sh" and (idx // 3) % arr.shape[1] >= (g["sh_degree"] + 1) ** 2:
                continue
            step = h * max(1.0, abs(float(arr.reshape(-1)[idx])))
            f1, s1 = central(key, idx, step)
            f2, s2 = central(key, idx, step / 2)
            if not (s1 and s2):
                continue  # a discrete decision flipped: the loss is not smooth here
            fd = (4 * f2 - f1) / 3
            tol = atol + rtol * max(abs(fd), abs(ana[idx]))
            assert abs(fd - ana[idx]) <= tol, (key, idx, fd, ana[idx], f1, f2)
            checked += 1
    return checked


def _fd_scene(seed, P=6, sh_degree=3, W=24, H=20, V=2):
    rng = np.random.default_rng(seed)
    means = rng.uniform(-0.3, 0.3, (P, 3))
    g = scene(means, log_scales=rng.uniform(-2.6, -1.8, (P, 3)), quats=rng.normal(size=(P, 4)),
              logits=rng.uniform(-1, 1.5, P), sh=rng.normal(0, 0.4, (P, (sh_degree + 1) ** 2, 3)),
              sh_degree=sh_degree)
    cams = synth.cams_array([synth.look_at([2.0 * math.cos(a), 2.0 * math.sin(a), 0.6], [0, 0, 0], W, H, 0.9 * W)
                             for a in np.linspace(0.3, 2.0, V)])
    dL = rng.normal(0, 1, (V, 3, H, W)).astype(np.float32)
    return g, cams, dL


@pytest.mark.parametrize("seed", [0, 1])
def test_P10_all_gradients_match_finite_differences(seed):
    """Every parameter gradient (means, log-scales, quaternion incl. normalisation,
    opacity logit, SH deg 3) = central FD of L = Σ ∂L/∂C · C, in fp64,
    with a non-zero background so the T_final·bg term is exercised (R16)."""
    g, cams, dL = _fd_scene(seed)
    n = _fd_check(g, cams, dL, bg=(0.2, 0.5, 0.1))
    assert n > 200


def test_P10_fd_with_jacobian_clamp():
    """A Gaussian far off-screen where ũx is clamped (R4: exact zero through the clamp,
    k=1 in ∂J/∂t.z) — FD agrees with the exact clamp gradient."""
    W = H = 24
    g = scene([[1.6, 0.0, 2.0], [0.2, 0.1, 2.5]], log_scales=np.full((2, 3), -0.7),
              logits=[2.0, 1.0], sh=np.full((2, 1, 3), 0.5))
    cams = synth.cams_array([synth.make_camera(np.eye(3), [0, 0, 0], W, H, 0.9 * W)])
    o = oracle.Oracle(g, cams)
    p = o.pairs()
    assert p["vis"][0, 0] == 1 and 1.6 / 2.0 > 0.65 * W / (0.9 * W)  # ux beyond the clamp limit
    dL = np.random.default_rng(3).normal(0, 1, (1, 3, H, W)).astype(np.float32)
    assert _fd_check(g, cams, dL) > 20


def test_P9_linearity():
    """dL ≡ 0 → every gradient and E is 0; dL → 2·dL doubles them exactly."""
    g, cams, dL = _fd_scene(5)
    o = oracle.Oracle(g, cams)
    z = o.backward(np.zeros_like(dL))
    assert all(np.all(v == 0) for k, v in z.items() if k != "vis")
    a = o.backward(dL)
    b = o.backward(2 * dL)
    for k in a:
        if k != "vis":
            np.testing.assert_array_equal(b[k], 2 * a[k])


# -------------------------------------------------------------------- ADC
def test_P11_adc_golden_examples():
    for line in open(os.path.join(GOLDEN, "adc_examples.txt")):
        if not line.strip() or line.startswith("#"):
            continue
        name, v, gx, gy, exp = [s.strip() for s in line.split("|")]
        out = oracle.adc_example([int(x) for x in v.split(",")], [float(x) for x in gx.split(",")],
                                 [float(x) for x in gy.split(",")])
        np.testing.assert_allclose(out, [float(x) for x in exp.split()], atol=1e-12, err_msg=name)


def test_P12_ordering_and_single_view_collapse():
    """E1 ≥ E2 ≥ E_old for every Gaussian (triangle inequality); one view ⇒
    E2 = E_old exactly."""
    g, cams = synth.make_scene("tiny")
    dL = synth.make_dLdC_scaled(4, 64, 64, 1)
    gr = oracle.Oracle(g, cams).backward(dL)
    assert np.all(gr["e1"] >= gr["e2"] * (1 - 1e-12))
    assert np.all(gr["e2"] >= gr["e_old"] * (1 - 1e-12))
    assert np.any(gr["e1"] > 1.01 * gr["e2"]) and np.any(gr["e2"] > 1.01 * gr["e_old"])
    g1 = oracle.Oracle(g, cams[:1]).backward(dL[:1])
    np.testing.assert_array_equal(g1["e2"], g1["e_old"])
    assert g1["e2"].max() > 0


def test_E1_is_norm_and_add_per_pixel():
    """E1 = Σ over pixels of ‖∇_{p_i}L‖ ('norm and add'): the per-pair E1 of a
    full ∂L/∂C equals the sum of the E1's from each single pixel's ∂L/∂C, while the
    per-pair Σ∇ is additive (linearity)."""
    W = H = 8
    g = scene([[0.02, -0.01, 2.0], [0.0, 0.03, 2.4]], log_scales=np.full((2, 3), -2.2),
              logits=[0.5, 1.0], sh=np.full((2, 1, 3), 0.4))
    cams = synth.cams_array([synth.make_camera(np.eye(3), [0, 0, 0], W, H, 10.0)])
    dL = np.random.default_rng(0).normal(0, 1, (1, 3, H, W)).astype(np.float32)
    o = oracle.Oracle(g, cams)
    o.backward(dL)
    full = o.pair_grads()
    e1 = np.zeros(2)
    gs = np.zeros((2, 2))
    for y in range(H):
        for x in range(W):
            d = np.zeros_like(dL)
            d[0, :, y, x] = dL[0, :, y, x]
            o.backward(d)
            pg = o.pair_grads()[0]
            e1 += pg[:, 2]
            gs += pg[:, :2]
            np.testing.assert_allclose(pg[:, 2], np.hypot(pg[:, 0], pg[:, 1]), rtol=1e-12, atol=1e-300)
    np.testing.assert_allclose(full[0, :, 2], e1, rtol=1e-12)
    np.testing.assert_allclose(full[0, :, :2], gs, rtol=1e-9, atol=1e-12)
    assert np.all(full[0, :, 2] > np.hypot(full[0, :, 0], full[0, :, 1]) * 1.01)


def test_P13_b2_opposite_cameras_cancel():
    """Appendix B.2: Gaussian at the origin, opposite cameras (golden file),
    ∂L/∂C of view B = x-mirror of view A's → per-view Σ∇ are opposite in x, E_old ≈ 0 <
    E2 ≤ E1, while the world gradient is along x and both views add to it.  Also pins
    the NDC scale (R2): Σ∇_x = (∂L/∂μ_x)_view · z_cam/P0 with P0 = 2f/W."""
    rows = [l.split("|") for l in open(os.path.join(GOLDEN, "b2_cameras.txt")) if l.strip() and not l.startswith("#")]
    W = H = 33
    f = 30.0
    cams = synth.cams_array([synth.make_camera(np.array(r[1].split(), float).reshape(3, 3),
                                               np.array(r[2].split(), float), W, H, f) for r in rows])
    g = scene([0, 0, 0], log_scales=np.full(3, math.log(0.08)), logits=[1.0], sh=np.full((1, 1, 3), 0.7))
    xs = np.arange(W) - 16.0
    ramp = np.tile(np.sign(xs)[None, :] * (1 + 0.01 * np.abs(xs)[None, :]), (H, 1))
    dA = np.tile(ramp[None], (3, 1, 1))
    dL = np.stack([dA, dA[:, :, ::-1]]).astype(np.float32)
    o = oracle.Oracle(g, cams)
    gr = o.backward(dL)
    pg = o.pair_grads()[:, 0]
    assert abs(pg[0, 0]) > 0
    np.testing.assert_allclose(pg[1, 0], -pg[0, 0], rtol=1e-9)
    assert abs(pg[0, 1]) < 1e-9 * abs(pg[0, 0])
    assert gr["e_old"][0] < 1e-8 * gr["e2"][0]
    np.testing.assert_allclose(gr["e2"][0], 2 * abs(pg[0, 0]), rtol=1e-12)
    assert gr["e1"][0] >= gr["e2"][0]
    dm = gr["d_means"][0]
    assert abs(dm[0]) > 0 and abs(dm[1]) < 1e-9 * abs(dm[0]) and abs(dm[2]) < 1e-9 * abs(dm[0])
    # single view A: world x-gradient ↔ NDC x-gradient (isotropic on-axis ⇒ only μ' moves)
    oA = oracle.Oracle(g, cams[:1])
    gA = oA.backward(dL[:1])
    P0 = 2 * f / W
    np.testing.assert_allclose(oA.pair_grads()[0, 0, 0], gA["d_means"][0, 0] * 1.0 / P0, rtol=1e-9)


def test_P16_gid_permutation_invariance():
    """With distinct depths, relabelling the Gaussians changes nothing but the labels."""
    g, cams = synth.make_scene(synth.scaled(synth.CONFIGS["tiny"], P=400))
    dL = synth.make_dLdC_scaled(4, 64, 64, 7)
    perm = np.random.default_rng(1).permutation(400)
    gp = {k: (v[perm] if isinstance(v, np.ndarray) else v) for k, v in g.items()}
    a = oracle.Oracle(g, cams)
    b = oracle.Oracle(gp, cams)
    ga, gb = a.backward(dL), b.backward(dL)
    ia, ib = a.image(), b.image()
    np.testing.assert_array_equal(ia["n_contrib"], ib["n_contrib"])
    np.testing.assert_array_equal(ia["rgb"], ib["rgb"])
    for k in ga:
        np.testing.assert_allclose(gb[k], ga[k][perm], rtol=1e-12, atol=1e-15)


# ---------------------------------------------------------------------- SH
def _Y_textbook(k, d):
    """Real SH in the [3DGS] sign convention, written from the textbook normalisations
    (1/2)√(1/π), √(3/4π), (1/2)√(15/π), (1/4)√(5/π), (1/4)√(15/π), (1/4)√(35/2π),
    (1/2)√(105/π), (1/4)√(21/2π), (1/4)√(7/π)."""
    x, y, z = d
    pi = math.pi
    c = [0.5 * math.sqrt(1 / pi), math.sqrt(3 / (4 * pi))]
    t = {0: c[0], 1: -c[1] * y, 2: c[1] * z, 3: -c[1] * x,
         4: 0.5 * math.sqrt(15 / pi) * x * y, 5: -0.5 * math.sqrt(15 / pi) * y * z,
         6: 0.25 * math.sqrt(5 / pi) * (2 * z * z - x * x - y * y), 7: -0.5 * math.sqrt(15 / pi) * x * z,
         8: 0.25 * math.sqrt(15 / pi) * (x * x - y * y),
         9: -0.25 * math.sqrt(35 / (2 * pi)) * y * (3 * x * x - y * y), 10: 0.5 * math.sqrt(105 / pi) * x * y * z,
         11: -0.25 * math.sqrt(21 / (2 * pi)) * y * (4 * z * z - x * x - y * y),
         12: 0.25 * math.sqrt(7 / pi) * z * (2 * z * z - 3 * x * x - 3 * y * y),
         13: -0.25 * math.sqrt(21 / (2 * pi)) * x * (4 * z * z - x * x - y * y),
         14: 0.25 * math.sqrt(105 / pi) * z * (x * x - y * y),
         15: -0.25 * math.sqrt(35 / (2 * pi)) * x * (x * x - 3 * y * y)}
    return t[k]


def test_P17_sh_basis_along_axes_and_diagonal():
    """rgb = max(0, Σ_k Y_k(dir) sh_k + 0.5), dir from the camera centre (R17): one unit
    coefficient at a time, viewed along ±x, ±y, ±z and a diagonal."""
    dirs = [(1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1), (1, 2, 2)]
    for dvec in dirs:
        d = np.array(dvec, float) / np.linalg.norm(dvec)
        cam = synth.look_at(-2.5 * d, [0, 0, 0], 16, 16, 20.0)
        for k in range(16):
            sh = np.zeros((1, 16, 3))
            sh[0, k, :] = [0.3, -0.2, 0.1]
            g = scene([0, 0, 0], sh=sh, sh_degree=3)
            o = oracle.Oracle(g, synth.cams_array([cam]))
            dd = np.array([0, 0, 0]) - (-(np.array(cam["R"], np.float64).reshape(3, 3).T @ np.array(cam["t"], np.float64)))
            dd /= np.linalg.norm(dd)
            exp = np.maximum(0, _Y_textbook(k, dd) * np.array([0.3, -0.2, 0.1], np.float32).astype(float) + 0.5)
            np.testing.assert_allclose(o.pairs()["rgb"][0, 0], exp, atol=1e-7, err_msg=f"k={k} dir={dvec}")


def test_tile_mask_mode_equals_full_run_on_the_mask():
    """Masked oracle (used for sampled checks at full size): on the masked tiles it
    reproduces the full run exactly; with ∂L/∂C zero outside them, every gradient and
    E statistic equals the full run's."""
    g, cams = synth.make_scene(synth.scaled(synth.CONFIGS["tiny"], P=600))
    V, T = 4, 16
    rng = np.random.default_rng(2)
    mask = (rng.uniform(size=(V, T)) < 0.3).astype(np.uint8)
    mask[0, :] = 0
    mask[0, 5] = 1
    pix = np.zeros((V, 64, 64), bool)
    for v in range(V):
        for t in range(T):
            if mask[v, t]:
                pix[v, (t // 4) * 16:(t // 4) * 16 + 16, (t % 4) * 16:(t % 4) * 16 + 16] = True
    dL = synth.make_dLdC_scaled(V, 64, 64, 5) * pix[:, None]
    full = oracle.Oracle(g, cams)
    gf = full.backward(dL)
    imf = full.image()
    m = oracle.Oracle(g, cams, tile_mask=mask)
    gm = m.backward(dL)
    imm = m.image()
    np.testing.assert_array_equal(imm["n_contrib"][pix], imf["n_contrib"][pix])
    np.testing.assert_array_equal(imm["rgb"].transpose(0, 2, 3, 1)[pix], imf["rgb"].transpose(0, 2, 3, 1)[pix])
    for k in gf:
        np.testing.assert_allclose(gm[k], gf[k], rtol=1e-12, atol=1e-15, err_msg=k)
    off_f, gid_f = full.lists()
    off_m, gid_m = m.lists()
    for b in np.nonzero(mask.reshape(-1))[0]:
        np.testing.assert_array_equal(gid_m[off_m[b]:off_m[b + 1]], gid_f[off_f[b]:off_f[b + 1]])


def test_predicted_depth_single_gaussian():
    """NEXT-2 predicted depth Σ dᵢαᵢTᵢ: one Gaussian at depth z ⇒ z·α on its
    footprint, 0 elsewhere; two co-centred terms ⇒ z₁α₁ + z₂α₂(1−α₁)."""
    s, z, f, W = 0.06, 2.0, 40.0, 32
    g = scene([0, 0, z], log_scales=np.full(3, math.log(s)), logits=[0.3])
    o = oracle.Oracle(g, cam_identity(W=W, H=W, f=f))
    im = o.forward()
    np.testing.assert_allclose(o.depth()[0], z * (1 - im["T_final"][0]), atol=1e-12)
    g2 = scene([[0, 0, 2.0], [0, 0, 3.0]], log_scales=np.full((2, 3), math.log(0.05)), logits=[0.0, math.log(9.0)])
    o2 = oracle.Oracle(g2, cam_identity(W=33, H=33, f=40.0))
    o2.forward()
    assert abs(o2.depth()[0, 16, 16] - (2.0 * 0.5 + 3.0 * 0.9 * 0.5)) < 1e-6


# ---------------------------------------------- O1 general rotation, O2 off-axis EWA
def _rodrigues(axis, theta):
    """Rotation by θ about the unit axis n (Rodrigues): R = I + sinθ K + (1 − cosθ) K²,
    K the cross-product matrix of n — built without any quaternion formula."""
    n = np.asarray(axis, float) / np.linalg.norm(axis)
    K = np.array([[0, -n[2], n[1]], [n[2], 0, -n[0]], [-n[1], n[0], 0]])
    return np.eye(3) + math.sin(theta) * K + (1 - math.cos(theta)) * K @ K


def _quat_axis_angle(axis, theta):
    n = np.asarray(axis, float) / np.linalg.norm(axis)
    return np.concatenate([[math.cos(theta / 2)], math.sin(theta / 2) * n])


def _conic_to_cov(p, v=0, i=0):
    A, B, C = (float(p[k][v, i]) for k in ("A", "B", "C"))
    return np.linalg.inv(np.array([[A, B], [B, C]]))


ROT_CASES = [((1, 0, 0), math.radians(37)), ((0, 1, 0), math.radians(-61)), ((1, 2, -0.5), math.radians(113)),
             ((0.3, -1, 0.8), math.radians(-152))]


@pytest.mark.parametrize("axis,theta", ROT_CASES)
def test_P1b_rotation_matches_rodrigues_through_three_cameras(axis, theta):
    """O1 R(q) for general axes and angles: Σ = R S² Rᵀ with R from Rodrigues'
    axis–angle formula.  Three on-axis cameras looking along world z, x and y each see the
    2×2 block (f/z)²·(R_c Σ R_cᵀ)[:2,:2] + 0.3·I as the inverse conic (P3's EWA with ũ = 0),
    so together they fix all six entries of Σ.  A transposed R(q), or a sign error in an
    off-diagonal entry, changes Σ for every generic rotation here."""
    s = np.array([0.08, 0.03, 0.05])
    z, f, W = 2.0, 400.0, 64
    g = scene([0, 0, 0], log_scales=np.log(s), quats=_quat_axis_angle(axis, theta))
    Rs = [np.eye(3), np.array([[0, 1, 0], [0, 0, 1], [1, 0, 0]]), np.array([[0, 0, 1], [1, 0, 0], [0, 1, 0]])]
    cams = synth.cams_array([synth.make_camera(Rc, [0, 0, z], W, W, f) for Rc in Rs])
    o = oracle.Oracle(g, cams)
    p = o.pairs()
    s32 = np.exp(np.log(s).astype(np.float32).astype(np.float64))
    Rr = _rodrigues(axis, theta)
    Sig = Rr @ np.diag(s32 ** 2) @ Rr.T
    for v, Rc in enumerate(Rs):
        got = (_conic_to_cov(p, v) - 0.3 * np.eye(2)) / (f / z) ** 2
        ref = (Rc @ Sig @ Rc.T)[:2, :2]
        np.testing.assert_allclose(got, ref, rtol=0, atol=2e-5 * np.abs(ref).max(), err_msg=f"camera {v}")
    # the fp64 value chain (activate64/project64): the rendered α of the single Gaussian is
    # o·exp(−½ dᵀ Σ'⁻¹ d) with Σ' from the same independent Σ (camera 0, bg = 0, rgb = 1)
    g["sh"] = np.full((1, 1, 3), 0.5 / C0, np.float32)
    o = oracle.Oracle(g, cams[:1])
    im = o.forward()
    Sp = (f / z) ** 2 * Sig[:2, :2] + 0.3 * np.eye(2)
    Si = np.linalg.inv(Sp)
    c = (W - 1) / 2
    for (x, y) in [(31, 31), (28, 35), (36, 30), (33, 25)]:
        d = np.array([c - x, c - y])
        alpha = 0.5 * math.exp(-0.5 * d @ Si @ d)
        assert im["n_contrib"][0, y, x] == 1
        rgb1 = float(np.float32(0.5 / C0)) * C0 + 0.5
        assert abs(im["rgb"][0, 0, y, x] - rgb1 * alpha) <= 1e-7 * alpha, (x, y)  # fp32 inputs


def _pinhole(t, f, c):
    return np.array([f * t[0] / t[2] + c, f * t[1] / t[2] + c])


def _offaxis_case():
    s = np.array([0.012, 0.006, 0.04])  # elongated in its local z
    q = _quat_axis_angle((0.4, -0.7, 0.5), math.radians(71))
    Rc = _rodrigues((0.2, 1.0, -0.3), math.radians(24))  # generic camera rotation (W ≠ I)
    t_cam = np.array([0.7, -0.5, 2.0])  # off-axis: ux = 0.35, uy = −0.25 (inside the clamp)
    tv = np.array([0.1, 0.2, -0.3])
    mu = Rc.T @ (t_cam - tv)  # x_c = R μ + t  ⇒  μ = Rᵀ (x_c − t)
    return s, q, Rc, tv, mu


def test_P2b_offaxis_ewa_matches_pinhole_linearisation():
    """O2 off-axis EWA: Σ' = J W Σ Wᵀ Jᵀ + 0.3·I where J is the
    Jacobian of the pinhole map (x, y, z) ↦ (f x/z + c, f y/z + c) at the camera-space mean.
    Here J is taken by central finite differences of that map in fp64 (no formula shared
    with the oracle), W is the camera rotation and Σ comes from Rodrigues — off-axis
    (ux = 0.35, uy = −0.25) and with a depth-elongated Σ, so the J02/J12 column matters:
    flipping its sign moves Σ' by O(1)."""
    s, q, Rc, tv, mu = _offaxis_case()
    f, W = 50.0, 64
    c = (W - 1) / 2
    g = scene(mu, log_scales=np.log(s), quats=q)
    cam = synth.cams_array([synth.make_camera(Rc, tv, W, W, f)])
    p = oracle.Oracle(g, cam).pairs()
    t = Rc.astype(np.float32).astype(np.float64) @ mu.astype(np.float32).astype(np.float64) \
        + tv.astype(np.float32).astype(np.float64)
    h = 1e-6
    J = np.column_stack([(_pinhole(t + h * e, f, c) - _pinhole(t - h * e, f, c)) / (2 * h) for e in np.eye(3)])
    s32 = np.exp(np.log(s).astype(np.float32).astype(np.float64))
    Rr = _rodrigues((0.4, -0.7, 0.5), math.radians(71))
    Sig = Rr @ np.diag(s32 ** 2) @ Rr.T
    Wc = Rc.astype(np.float32).astype(np.float64)
    Sp = J @ Wc @ Sig @ Wc.T @ J.T + 0.3 * np.eye(2)
    got = _conic_to_cov(p)
    np.testing.assert_allclose(got, Sp, rtol=0, atol=3e-5 * np.abs(Sp).max())
    np.testing.assert_allclose([p["px"][0, 0], p["py"][0, 0]], _pinhole(t, f, c), rtol=0, atol=2e-4)
    # the fp64 value chain (project64): α of the rendered Gaussian at pixels near μ' is
    # o·exp(−½ dᵀ Σ'⁻¹ d), d = μ' − p, with the same independent Σ' and μ' = π(t)
    g["sh"] = np.full((1, 1, 3), 0.5 / C0, np.float32)
    im = oracle.Oracle(g, cam).forward()
    mp = _pinhole(t, f, c)
    Si = np.linalg.inv(Sp)
    rgb1 = float(np.float32(0.5 / C0)) * C0 + 0.5
    for (x, y) in [(int(mp[0]), int(mp[1])), (int(mp[0]) + 1, int(mp[1]) - 1), (int(mp[0]) - 1, int(mp[1]))]:
        d = mp - [x, y]
        alpha = 0.5 * math.exp(-0.5 * d @ Si @ d)
        assert im["n_contrib"][0, y, x] == 1
        assert abs(im["rgb"][0, 0, y, x] - rgb1 * alpha) <= 1e-6 * alpha, (x, y)
    # J's third column really contributes here (the pin is not blind to its sign)
    Jf = J.copy()
    Jf[:, 2] *= -1
    Spf = Jf @ Wc @ Sig @ Wc.T @ Jf.T + 0.3 * np.eye(2)
    assert np.abs(Spf - Sp).max() > 0.2 * np.abs(Sp - 0.3 * np.eye(2)).max()


def test_P2c_offaxis_ewa_monte_carlo():
    """The same off-axis projection checked against samples: points drawn from a small
    anisotropic Gaussian N(μ, Σ) (Σ from Rodrigues) are pushed through the exact pinhole
    map; their empirical 2-D covariance approaches J W Σ Wᵀ Jᵀ = Σ' − 0.3·I (the EWA
    first-order model) — within Monte-Carlo error plus the O(s/z) linearisation bias."""
    s, q, Rc, tv, mu = _offaxis_case()
    s = s / 4  # small footprint: linearisation bias ~ (s/z)²
    f, W = 50.0, 64
    c = (W - 1) / 2
    g = scene(mu, log_scales=np.log(s), quats=q)
    cam = synth.cams_array([synth.make_camera(Rc, tv, W, W, f)])
    p = oracle.Oracle(g, cam).pairs()
    got = _conic_to_cov(p) - 0.3 * np.eye(2)
    rng = np.random.default_rng(2506)
    n = 4_000_000
    Rr = _rodrigues((0.4, -0.7, 0.5), math.radians(71))
    s32 = np.exp(np.log(s).astype(np.float32).astype(np.float64))
    X = mu + (rng.standard_normal((n, 3)) * s32) @ Rr.T
    tc = X @ Rc.T + tv
    uv = np.column_stack([f * tc[:, 0] / tc[:, 2] + c, f * tc[:, 1] / tc[:, 2] + c])
    emp = np.cov(uv.T)
    np.testing.assert_allclose(got, emp, rtol=0, atol=5e-3 * np.abs(emp).max())


def test_P17b_sh_clamp_decision_is_the_sign_of_the_colour():
    """The SH clamp (rgb < 0 → 0, masked gradient; R17) is a decision, taken in fp32 CA
    (DESIGN.md §4.4): for random degree-3 coefficients and view directions its bits equal
    the sign of Σ_k Y_k(dir)·sh_k + 0.5 computed with the textbook basis in fp64, wherever
    that value is not within rounding of 0 (|v| > 1e-5)."""
    rng = np.random.default_rng(17)
    n = 600
    means = rng.uniform(-1, 1, (n, 3))
    sh = rng.normal(0, 0.5, (n, 16, 3)).astype(np.float32)
    sh[:, 0, :] = rng.normal(-0.9, 0.6, (n, 3))  # many colours near and below 0
    g = scene(means, log_scales=np.full((n, 3), -4.0), sh=sh, sh_degree=3)
    cams = [synth.look_at(np.array(e), [0, 0, 0], 64, 64, 50.0) for e in ([4, 1, 2], [-3, 3, 1], [0.5, -4, 3])]
    o = oracle.Oracle(g, synth.cams_array(cams))
    p = o.pairs()
    seen = 0
    for v, cam in enumerate(cams):
        Rv = np.array(cam["R"], np.float64).reshape(3, 3)
        cpos = -Rv.T @ np.array(cam["t"], np.float64)
        for i in np.nonzero(p["vis"][v])[0]:
            d = means[i].astype(np.float32).astype(np.float64) - cpos
            d /= np.linalg.norm(d)
            Y = np.array([_Y_textbook(k, d) for k in range(16)])
            val = Y @ sh[i].astype(np.float64) + 0.5
            ok = np.abs(val) > 1e-5
            bits = (p["clamp"][v, i] >> np.arange(3)) & 1
            np.testing.assert_array_equal(bits[ok], (val < 0)[ok].astype(int), err_msg=f"view {v} gid {i}")
            seen += int(np.sum(val < 0))
    assert seen > 100  # the clamp is exercised


# ------------------------------------------------------- fp32 canonical-arithmetic image (§5)
def test_image32_is_the_fp32_evaluation_of_the_fp64_image():
    """image32 (the decisions' T and α, C = fma(rgb32, α·T, C)) against the fp64 value chain:
    within 1e-5 + 2^-24 per walked entry, and the deviation is carried by the fp32 alphas —
    an fp64 chain fed the fp32 alphas (rgb_x) deviates as much (R47)."""
    import dataclasses
    cfg = dataclasses.replace(synth.CONFIGS["tiny"], P=20_000)
    g, cams = synth.make_scene(cfg)
    o = oracle.Oracle(g, cams, bg=(0.1, 0.2, 0.3))
    im = o.forward()
    i32 = o.image32()
    n = im["n_contrib"].astype(np.float64)
    assert n.max() > 100
    d32 = np.abs(i32["rgb"].astype(np.float64) - im["rgb"])
    dx = np.abs(i32["rgb_x"] - im["rgb"])
    assert np.all(d32 <= 1e-5 + 2.0 ** -24 * n[:, None])
    assert np.all(np.abs(i32["T_final"] - im["T_final"]) <= 1e-5 + 2.0 ** -24 * n)
    assert dx.max() >= 0.5 * d32.max() > 0
    # the single-Gaussian case is exact up to the fp32 colour and α: rgb32·α + (1 − α)·bg
    g1 = dict(means=np.zeros((1, 3), np.float32), log_scales=np.full((1, 3), np.log(0.2), np.float32),
              quats=np.array([[1, 0, 0, 0]], np.float32), opacity_logits=np.array([1.0], np.float32),
              sh=np.array([[[0.3, -0.2, 0.5]]], np.float32), sh_degree=0)
    cam = synth.cams_array([synth.make_camera(np.eye(3), [0, 0, 2.0], 32, 32, 40.0)])
    o1 = oracle.Oracle(g1, cam)
    im1 = o1.forward()
    np.testing.assert_allclose(o1.image32()["rgb"], im1["rgb"], atol=2e-7)


def test_threads_change_no_result():
    """oracle-mt (the timing baseline): lists, images, decisions identical, and the per-pair /
    per-Gaussian sums equal to fp64 reordering."""
    import dataclasses
    cfg = dataclasses.replace(synth.CONFIGS["tiny"], P=3000, sh_degree=0)
    g, cams = synth.make_scene(cfg)
    dL = synth.make_dLdC_scaled(cfg.V, cfg.H, cfg.W, 1)
    res = []
    for n in (1, 4):
        oracle.set_threads(n)
        try:
            o = oracle.Oracle(g, cams, bg=(0.1, 0.2, 0.3))
            r = o.backward(dL)
            res.append((o.lists(), o.image(), o.decision_hash(), r))
        finally:
            oracle.set_threads(1)
    (l1, i1, h1, r1), (l4, i4, h4, r4) = res
    for a, b in zip(l1, l4):
        np.testing.assert_array_equal(a, b)
    for k in i1:
        np.testing.assert_array_equal(i1[k], i4[k])
    assert h1 == h4
    for k in r1:
        np.testing.assert_allclose(r4[k], r1[k], rtol=1e-12, atol=1e-12 * max(1e-300, np.abs(r1[k]).max()))
