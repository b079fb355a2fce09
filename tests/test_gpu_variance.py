"""NEXT-4 parity: the variance lab through the C ABI (mvgs_loss_grad / mvgs_grad_moments /
mvgs_grad_variance and the S1–S8 gradient engine) against oracle/variance.py.
Kernels vs fp64 numpy: ℓ2 gradient bit-exact (same fp32 operations), sums rel 1e-12.  Lab vs
oracle: 𝕍 rel 2e-3 (per-element gradient tolerance of §5 carried through a difference of
two sums); lab vs the textbook finite-population law on the GPU's own per-view gradients:
rel 1e-5 (view independence of the rasterizer)."""
import itertools

import numpy as np
import pytest
import torch

import synth
from gpu_harness import to_dev
from oracle import variance as ov

pytestmark = pytest.mark.gpu


def test_moment_and_variance_kernels(require_gpu):
    from paper_2506_12727_b200 import mvgs
    rng = np.random.default_rng(0)
    n, K = 1_000_003, 5
    gs = (rng.normal(size=(K, n)) + 0.3).astype(np.float32)
    ctx = mvgs.create(0)
    try:
        s = torch.zeros(n, dtype=torch.float64, device="cuda")
        ss = torch.zeros(1, dtype=torch.float64, device="cuda")
        out = torch.zeros(1, dtype=torch.float64, device="cuda")
        for k in range(K):
            mvgs.grad_moments(ctx, torch.from_numpy(gs[k]).cuda(), s, ss)
        mvgs.grad_variance(ctx, s, ss, K, out)
        torch.cuda.synchronize()
        msq, _, v = ov.estimator(gs.astype(np.float64))
        np.testing.assert_allclose(s.cpu().numpy(), gs.astype(np.float64).sum(0), rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(float(ss) / K, msq, rtol=1e-12)
        np.testing.assert_allclose(float(out), v, rtol=1e-9)
    finally:
        mvgs.destroy(ctx)


@pytest.mark.parametrize("mode", [0, 1])
def test_loss_grad_kernel(require_gpu, mode):
    from paper_2506_12727_b200 import mvgs
    rng = np.random.default_rng(1)
    a = rng.uniform(0, 1, 777_777).astype(np.float32)
    b = rng.uniform(0, 1, 777_777).astype(np.float32)
    b[:100] = a[:100]  # exact ties: ℓ1 gradient 0
    ctx = mvgs.create(0)
    try:
        dL = torch.empty(a.size, device="cuda")
        loss = torch.zeros(1, dtype=torch.float64, device="cuda")
        sc = np.float32(1.0 / a.size)
        mvgs.loss_grad(ctx, torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), dL, mode, float(sc), loss)
        torch.cuda.synchronize()
        d = a - b
        ref = np.sign(d) * sc if mode == 0 else np.float32(2.0) * sc * d
        np.testing.assert_array_equal(dL.cpu().numpy(), ref.astype(np.float32))
        lref = np.abs(d.astype(np.float64)).sum() if mode == 0 else (d.astype(np.float64) ** 2).sum()
        np.testing.assert_allclose(float(loss), lref, rtol=1e-12)
    finally:
        mvgs.destroy(ctx)


@pytest.mark.parametrize("mode", [0, 1])
def test_loss_grad_u8_target(require_gpu, mode):
    """mvgs_loss_grad_u8: an 8-bit target t is the fp32 value t·fl(1/255); the result equals the
    fp32 entry point's on that target exactly (gradient and loss)."""
    from paper_2506_12727_b200 import mvgs
    rng = np.random.default_rng(2)
    n = 500_003
    t8 = rng.integers(0, 256, n).astype(np.uint8)
    tf = t8.astype(np.float32) * np.float32(1.0 / 255.0)
    a = rng.uniform(0, 1, n).astype(np.float32)
    a[:64] = tf[:64]  # exact ties
    ctx = mvgs.create(0)
    try:
        sc = float(np.float32(1.0 / n))
        out = []
        for tgt in (torch.from_numpy(t8).cuda(), torch.from_numpy(tf).cuda()):
            dL = torch.empty(n, device="cuda")
            loss = torch.zeros(1, dtype=torch.float64, device="cuda")
            mvgs.loss_grad(ctx, torch.from_numpy(a).cuda(), tgt, dL, mode, sc, loss)
            torch.cuda.synchronize()
            out.append((dL.cpu().numpy(), float(loss)))
        np.testing.assert_array_equal(out[0][0], out[1][0])
        assert out[0][1] == out[1][1]
        d = a - tf
        ref = np.sign(d) * np.float32(sc) if mode == 0 else np.float32(2.0) * np.float32(sc) * d
        np.testing.assert_array_equal(out[0][0], ref.astype(np.float32))
    finally:
        mvgs.destroy(ctx)


def test_render_bwd_l1_equals_loss_kernel_then_backward(require_gpu):
    """mvgs_render_bwd_l1 (the ℓ1 loss of 8-bit targets fused into S7) against
    mvgs_loss_grad_u8 + mvgs_render_bwd on the same render: the same ∂L/∂C per pixel, so the
    parameter gradients and E statistics agree to the atomics' summation order, and the loss
    to the order of its per-warp double sums."""
    from paper_2506_12727_b200 import mvgs
    cfg = synth.scaled(synth.CONFIGS["garden"], P=20_000, V=3, W=173, H=131)
    g, cams = synth.make_scene(cfg)
    gd = to_dev(g)
    rng = np.random.default_rng(5)
    tgt = torch.from_numpy(rng.integers(0, 256, (3, 3, 131, 173), dtype=np.uint8)).cuda()
    R = mvgs.Rasterizer(0)
    out = {}
    for fused in (False, True):
        R.preprocess(gd, cams)
        rgb, Tf, nc = R.forward()
        loss = torch.zeros(1, dtype=torch.float64, device="cuda")
        grads, adc = R.alloc_backward()
        if fused:
            mvgs.render_bwd_l1(R.ctx, rgb, tgt, Tf, nc, loss=loss)
        else:
            dL = torch.empty_like(rgb)
            mvgs.loss_grad(R.ctx, rgb, tgt, dL, mvgs.LOSS_L1, loss=loss)
            mvgs.render_bwd(R.ctx, dL, Tf, nc)
        mvgs.adc_stats(R.ctx, grads, adc)
        torch.cuda.synchronize()
        out[fused] = ({k: v.cpu().numpy().astype(np.float64) for k, v in {**grads, **adc}.items()}, float(loss))
    a, b = out[False], out[True]
    assert abs(a[1] - b[1]) <= 1e-12 * abs(a[1])
    for k in a[0]:
        x, y = a[0][k], b[0][k]
        assert np.linalg.norm(x - y) <= 1e-5 * max(np.linalg.norm(x), 1e-30), k


@pytest.fixture(scope="module")
def lab_scene(require_gpu):
    M, W, H = 5, 64, 48
    cfg = synth.scaled(synth.CONFIGS["garden"], P=3000, V=M, W=W, H=H)
    g, cams = synth.make_scene(cfg)
    targets = synth.make_lab_targets(M, H, W, 7)
    return g, cams, targets


def test_lab_matches_oracle_and_finite_population_law(lab_scene):
    from paper_2506_12727_b200.lab import VarianceLab
    g, cams, targets = lab_scene
    M = len(cams)
    lab = VarianceLab(to_dev(g), cams, torch.from_numpy(targets).cuda())
    per_view = np.stack([lab.batch_gradient([i])["d_means"].reshape(-1).double().cpu().numpy() for i in range(M)])
    ref_pv = ov.view_gradients(g, cams, targets)
    for m in (1, 2, 3):
        batches = list(itertools.combinations(range(M), m))
        v_gpu = lab.run(batches)
        _, _, v_ref = ov.lab(g, cams, targets, batches)
        np.testing.assert_allclose(v_gpu, v_ref, rtol=2e-3)
        np.testing.assert_allclose(v_gpu, ov.finite_population_variance(per_view, m), rtol=1e-5)
        np.testing.assert_allclose(v_ref, ov.finite_population_variance(ref_pv, m), rtol=1e-9)


def test_multi_view_batches_have_lower_variance(lab_scene):
    """Fig. 3's ordering on the synthetic scene: 𝕍(B = 4) < 𝕍(B = 1)."""
    from paper_2506_12727_b200.lab import VarianceLab
    g, cams, targets = lab_scene
    lab = VarianceLab(to_dev(g), cams, torch.from_numpy(targets).cuda())
    rng = np.random.default_rng(3)
    v1 = lab.run([[int(rng.integers(5))] for _ in range(40)])
    v4 = lab.run([list(rng.choice(5, 4, replace=False)) for _ in range(40)])
    assert v4 < v1
