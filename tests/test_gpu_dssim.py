"""NEXT-2 parity: the 3D distance-aware D-SSIM through the C ABI
against oracle/dssim.py, and the renderer's predicted depth against the
oracle rasterizer's.  Tolerances: loss |Δ| ≤ 1e-5 (a mean of
fp32 SSIM values summed in fp64); gradient per tensor ‖Δ‖/‖ref‖ ≤ 1e-3 and per element
|Δ| ≤ 1e-3·|ref| + 1e-5·max|ref| (the main rule's relative part; the floor absorbs fp32
moments — variance by cancellation — and the hardware exp; measured need 1.8e-6, tensor
error 4e-6, scripts/dssim_err_probe.py);
depth |Δ| ≤ 2e-5·max depth (same decisions as the image, fp32 sum)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_harness import to_dev
from oracle import dssim

pytestmark = pytest.mark.gpu


def gpu_dssim(img, tgt, depth, Tf, cams, sigma=1.5, grad=True):
    from paper_2506_12727_b200 import mvgs
    dev = torch.device("cuda")
    ctx = mvgs.create(0)
    try:
        t = [torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (img, tgt, depth, Tf)]
        loss = torch.zeros(1, device=dev)
        g = torch.empty_like(t[0]) if grad else None
        mvgs.dssim3d(ctx, cams, *t, loss, g, sigma)
        torch.cuda.synchronize()
        return float(loss.item()), (g.cpu().numpy() if grad else None)
    finally:
        mvgs.destroy(ctx)


def check_grad(g, ref):
    rel = np.linalg.norm(g - ref) / np.linalg.norm(ref)
    assert rel <= 1e-3, rel
    tol = 1e-3 * np.abs(ref) + 1e-5 * np.max(np.abs(ref))
    bad = np.abs(g - ref) > tol
    assert not bad.any(), f"{bad.sum()} elements out of tolerance, max |Δ| {np.max(np.abs(g - ref)):.3e}"


@pytest.mark.parametrize("shape", [(2, 45, 61), (1, 16, 16), (1, 7, 5)])
def test_dssim3d_matches_oracle(require_gpu, shape):
    V, H, W = shape
    img, tgt, depth, Tf, cams = synth.make_dssim_inputs(V, H, W, seed=H + W)
    loss, g = gpu_dssim(img, tgt, depth, Tf, cams)
    ref_loss, ref_g = dssim.dssim3d(img, tgt, depth, Tf, cams)
    assert abs(loss - ref_loss) <= 1e-5, (loss, ref_loss)
    check_grad(g, ref_g)


def test_dssim3d_loss_only_and_sigma(require_gpu):
    img, tgt, depth, Tf, cams = synth.make_dssim_inputs(1, 33, 40, seed=3)
    loss, _ = gpu_dssim(img, tgt, depth, Tf, cams, sigma=2.5, grad=False)
    ref_loss, _ = dssim.dssim3d(img, tgt, depth, Tf, cams, sigma_px=2.5, grad=False)
    assert abs(loss - ref_loss) <= 1e-5


def test_dssim3d_more_views_than_one_launch(require_gpu):
    """V = 67 > 64 views per launch: view chunking keeps every view's intrinsics."""
    img, tgt, depth, Tf, cams = synth.make_dssim_inputs(67, 12, 14, seed=9)
    cams["fx"] *= np.linspace(0.5, 2.0, 67).astype(np.float32)
    loss, g = gpu_dssim(img, tgt, depth, Tf, cams)
    ref_loss, ref_g = dssim.dssim3d(img, tgt, depth, Tf, cams)
    assert abs(loss - ref_loss) <= 1e-5
    check_grad(g, ref_g)


def test_dssim3d_planar_equals_2d_ssim(require_gpu):
    """Fronto-parallel foreground plane: the GPU loss equals an independent 2D SSIM."""
    rng = np.random.default_rng(4)
    H, W = 30, 37
    img, tgt = rng.uniform(0, 1, (1, 3, H, W)).astype(np.float32), rng.uniform(0, 1, (1, 3, H, W)).astype(np.float32)
    depth = np.full((1, H, W), 3.25, np.float32)
    cams = synth.cams_array([synth.make_camera(np.eye(3), [0, 0, 0], W, H, 31.0)])
    loss, _ = gpu_dssim(img, tgt, depth, np.zeros((1, H, W), np.float32), cams, grad=False)
    ref = 1.0 - np.mean(dssim.ssim2d(img[0].astype(np.float64), tgt[0].astype(np.float64)))
    assert abs(loss - ref) <= 1e-5


def test_dssim3d_identical_images(require_gpu):
    img, _, depth, Tf, cams = synth.make_dssim_inputs(1, 20, 24, seed=5)
    loss, g = gpu_dssim(img, img, depth, Tf, cams)
    assert abs(loss) <= 1e-6 and np.max(np.abs(g)) <= 1e-7


def test_dssim3d_invalid_arguments(require_gpu):
    from paper_2506_12727_b200 import mvgs
    img, tgt, depth, Tf, cams = synth.make_dssim_inputs(1, 8, 8, seed=1)
    dev = torch.device("cuda")
    t = [torch.from_numpy(a).to(dev) for a in (img, tgt, depth, Tf)]
    loss = torch.zeros(1, device=dev)
    ctx = mvgs.create(0)
    try:
        with pytest.raises(mvgs.MvgsError):
            mvgs.dssim3d(ctx, cams, *t, loss, None, sigma_px=0.0)
        bad = cams.copy()
        bad["fx"] = 0
        with pytest.raises(mvgs.MvgsError):
            mvgs.dssim3d(ctx, bad, *t, loss, None)
    finally:
        mvgs.destroy(ctx)


def test_render_depth_matches_oracle(require_gpu):
    """Predicted depth Σ dᵢαᵢTᵢ of the renderer vs the oracle rasterizer; colour
    and T unchanged by the depth output."""
    from paper_2506_12727_b200 import mvgs
    cfg = synth.scaled(synth.CONFIGS["garden"], P=20_000, V=3, W=150, H=101)
    g, cams = synth.make_scene(cfg)
    o = oracle.Oracle(g, cams)
    o.forward()
    ref_d = o.depth()
    im = o.image()
    R = mvgs.Rasterizer(0)
    R.preprocess(to_dev(g), cams)
    rgb, Tf, nc = R.alloc_forward()
    d = torch.empty_like(Tf)
    mvgs.render_fwd_depth(R.ctx, rgb, Tf, nc, d)
    torch.cuda.synchronize()
    d = d.cpu().numpy()
    np.testing.assert_array_equal(nc.cpu().numpy(), im["n_contrib"])
    assert np.max(np.abs(rgb.cpu().numpy() - im["rgb"])) <= 1e-5
    assert np.max(np.abs(d - ref_d)) <= 2e-5 * np.max(np.abs(ref_d))
    del R
