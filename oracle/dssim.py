"""Oracle for NEXT-2: the 3D distance-aware D-SSIM loss.
TEST INFRASTRUCTURE ONLY (same import rules as oracle/__init__.py).

Definitions followed, in fp64, in the paper's notation:
  SSIM(I1, I2) = (2μ1μ2 + C1)(2τ12 + C2) / ((μ1² + μ2² + C1)(τ1² + τ2² + C2))
  μ1 = ⟨I1, K⟩, τ1² = ⟨I1∘I1, K⟩ − μ1², τ12 = ⟨I1∘I2, K⟩ − μ1μ2
  K*_σ(u, v) ∝ exp(−(X² + Y² + Z²)/2σ²), (X, Y, Z) the 3D point of window pixel
  (u, v) relative to the window centre's point, from the predicted depth
  D-SSIM = 1 − SSIM, averaged over window centres and colour channels.

Readings: 11×11 windows (radius 5), C1 = 0.01², C2 = 0.03²; the
kernel is renormalised to Σ = 1 over the window's in-image, non-background pixels;
a pixel is background when its T_final > 0.999; a background centre uses the
plain 2D Gaussian kernel (σ = sigma_px) over its whole window; σ3d at a centre c =
sigma_px · depth_c / fx, so a fronto-parallel plane reproduces the 2D kernel;
3D points are camera-space (x − cx)/fx·d, (y − cy)/fy·d, d — distances are
rotation-invariant, so this equals the paper's world-space kernel for one view;
depth is a constant of the loss (no gradient through the kernel weights).
"""
from __future__ import annotations

import numpy as np

C1 = 0.01 ** 2
C2 = 0.03 ** 2
RADIUS = 5


def _points(depth, cam):
    H, W = depth.shape
    y, x = np.mgrid[0:H, 0:W].astype(np.float64)
    d = depth.astype(np.float64)
    return np.stack([(x - float(cam["cx"])) / float(cam["fx"]) * d, (y - float(cam["cy"])) / float(cam["fy"]) * d, d], -1)


def window_weights(depth, T_final, cam, sigma_px=1.5, radius=RADIUS):
    """Normalised kernel K*[c, offset] for every centre c of one view: array
    [H, W, 2r+1, 2r+1] (zero outside the image / on excluded pixels)."""
    H, W = depth.shape
    X = _points(depth, cam)
    bg = T_final > 0.999
    k = 2 * radius + 1
    Wt = np.zeros((H, W, k, k))
    sig3 = sigma_px * depth.astype(np.float64) / float(cam["fx"])
    for dy in range(-radius, radius + 1):
        for dx in range(-radius, radius + 1):
            ys, xs = np.mgrid[0:H, 0:W]
            yy, xx = ys + dy, xs + dx
            inside = (yy >= 0) & (yy < H) & (xx >= 0) & (xx < W)
            yyc, xxc = np.clip(yy, 0, H - 1), np.clip(xx, 0, W - 1)
            d2 = np.sum((X[yyc, xxc] - X) ** 2, -1)
            w3 = np.exp(-d2 / (2 * np.maximum(sig3, 1e-30) ** 2)) * (~bg[yyc, xxc])
            w2 = np.exp(-(dx * dx + dy * dy) / (2 * sigma_px ** 2)) * np.ones((H, W))
            w = np.where(bg, w2, w3) * inside
            Wt[:, :, dy + radius, dx + radius] = w
    Wt /= Wt.sum(axis=(2, 3), keepdims=True)
    return Wt


def _gather(img, radius=RADIUS):
    """[C, H, W] → [C, H, W, 2r+1, 2r+1] window values (edge-clamped; weights zero them)."""
    C, H, W = img.shape
    k = 2 * radius + 1
    out = np.zeros((C, H, W, k, k))
    ys, xs = np.mgrid[0:H, 0:W]
    for dy in range(-radius, radius + 1):
        for dx in range(-radius, radius + 1):
            yy, xx = np.clip(ys + dy, 0, H - 1), np.clip(xs + dx, 0, W - 1)
            out[:, :, :, dy + radius, dx + radius] = img[:, yy, xx]
    return out


def dssim3d(img, target, depth, T_final, cams, sigma_px=1.5, radius=RADIUS, grad=True):
    """Loss and ∂loss/∂img for a batch: img, target [V,3,H,W]; depth, T_final [V,H,W]."""
    img = np.asarray(img, np.float64)
    target = np.asarray(target, np.float64)
    V, C, H, W = img.shape
    N = V * C * H * W
    total = 0.0
    g = np.zeros_like(img)
    for v in range(V):
        K = window_weights(depth[v], T_final[v], cams[v], sigma_px, radius)
        I1 = _gather(img[v], radius)
        I2 = _gather(target[v], radius)
        mu1 = np.sum(K * I1, axis=(3, 4))
        mu2 = np.sum(K * I2, axis=(3, 4))
        m11 = np.sum(K * I1 * I1, axis=(3, 4))
        m22 = np.sum(K * I2 * I2, axis=(3, 4))
        m12 = np.sum(K * I1 * I2, axis=(3, 4))
        s11, s22, s12 = m11 - mu1 ** 2, m22 - mu2 ** 2, m12 - mu1 * mu2
        A1, A2 = 2 * mu1 * mu2 + C1, 2 * s12 + C2
        B1, B2 = mu1 ** 2 + mu2 ** 2 + C1, s11 + s22 + C2
        S = A1 * A2 / (B1 * B2)
        total += np.sum(S)
        if not grad:
            continue
        # ∂S/∂m1, ∂S/∂m11, ∂S/∂m12 (raw moments), then scatter through the weights
        dS_m1 = S * (2 * mu2 / A1 - 2 * mu1 / B1) + (-S / B2) * (-2 * mu1) + (2 * S / A2) * (-mu2)
        dS_m11 = -S / B2
        dS_m12 = 2 * S / A2
        ys, xs = np.mgrid[0:H, 0:W]
        for dy in range(-radius, radius + 1):
            for dx in range(-radius, radius + 1):
                yy, xx = ys + dy, xs + dx
                ok = (yy >= 0) & (yy < H) & (xx >= 0) & (xx < W)
                w = K[:, :, dy + radius, dx + radius] * ok
                for ch in range(C):
                    contrib = w * (dS_m1[ch] + 2 * dS_m11[ch] * I1[ch, :, :, dy + radius, dx + radius]
                                   + dS_m12[ch] * I2[ch, :, :, dy + radius, dx + radius])
                    np.add.at(g[v, ch], (yy[ok], xx[ok]), contrib[ok])
    loss = 1.0 - total / N
    return loss, (-g / N if grad else None)


def ssim2d(img, target, sigma_px=1.5, radius=RADIUS):
    """Plain windowed SSIM with a truncated, renormalised 2D Gaussian kernel."""
    img = np.asarray(img, np.float64)
    target = np.asarray(target, np.float64)
    C, H, W = img.shape
    k = 2 * radius + 1
    off = np.arange(-radius, radius + 1)
    base = np.exp(-(off[:, None] ** 2 + off[None, :] ** 2) / (2 * sigma_px ** 2))
    ys, xs = np.mgrid[0:H, 0:W]
    K = np.zeros((H, W, k, k))
    for a, dy in enumerate(off):
        for b, dx in enumerate(off):
            ok = (ys + dy >= 0) & (ys + dy < H) & (xs + dx >= 0) & (xs + dx < W)
            K[:, :, a, b] = base[a, b] * ok
    K /= K.sum(axis=(2, 3), keepdims=True)
    I1, I2 = _gather(img, radius), _gather(target, radius)
    mu1, mu2 = np.sum(K * I1, axis=(3, 4)), np.sum(K * I2, axis=(3, 4))
    s11 = np.sum(K * I1 * I1, axis=(3, 4)) - mu1 ** 2
    s22 = np.sum(K * I2 * I2, axis=(3, 4)) - mu2 ** 2
    s12 = np.sum(K * I1 * I2, axis=(3, 4)) - mu1 * mu2
    return ((2 * mu1 * mu2 + C1) * (2 * s12 + C2)) / ((mu1 ** 2 + mu2 ** 2 + C1) * (s11 + s22 + C2))
