"""mvgs-synth v1 — seeded synthetic scenes, cameras and dL/dC for mvgs.

This module is the ONLY code shared by the CUDA path (bench, GPU tests) and the
oracle (CPU tests). It holds none of the method's arithmetic: it draws random
Gaussian parameters, places pinhole cameras and draws a per-pixel loss
gradient. Everything the rasterizer computes from these inputs is done
independently by `oracle/` and by `paper_2506_12727_b200/csrc/`.

Recipes follow SURVEY.md §8(d) M2 (the paper gives only dataset names,
PAPER.md:211; shapes and distributions are this build's proposal, recorded in
DESIGN.md §6):

* ``tiny``     — SPEC.md make_synthetic "orbit": 1,000 Gaussians in
                 the unit ball, SH degree 0, 4 cameras on a radius-3 circle,
                 64×64.
* ``object360``— Mip-NeRF-360-like: ground disc + central ellipsoid shell +
                 background cylinder (75 % surface Gaussians, flattened along
                 the surface normal) + 25 % volume Gaussians; cameras on a ring
                 looking at the centre.
* ``indoor``   — Deep-Blending-playroom-like: inner faces of a 6×8×3 room plus
                 12 random boxes; cameras inside looking outward.

All draws use ``numpy.random.Generator(PCG64(seed))`` in a fixed order.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

# Camera record, byte-identical to `mvgs_camera` (include/mvgs.h) and to the
# oracle's own `og_cam` (oracle/oracle.c): 19 four-byte fields, 76 bytes.
CAM_DTYPE = np.dtype(
    [
        ("R", "<f4", (9,)),  # world->camera rotation, row-major, x_c = R x + t
        ("t", "<f4", (3,)),
        ("fx", "<f4"),
        ("fy", "<f4"),
        ("cx", "<f4"),
        ("cy", "<f4"),
        ("width", "<i4"),
        ("height", "<i4"),
        ("znear", "<f4"),
    ]
)
assert CAM_DTYPE.itemsize == 76

SH_C0 = 0.28209479177387814  # only used to map a target colour to sh0 (input recipe)


@dataclass(frozen=True)
class Config:
    name: str
    P: int
    sh_degree: int
    V: int
    W: int
    H: int
    seed: int
    layout: str


CONFIGS = {
    "tiny": Config("tiny", 1_000, 0, 4, 64, 64, 1, "tiny"),
    "garden": Config("garden", 3_000_000, 3, 4, 1237, 822, 2, "object360"),
    "train": Config("train", 1_100_000, 3, 8, 980, 545, 3, "object360x"),
    "playroom": Config("playroom", 2_500_000, 3, 8, 1264, 832, 4, "indoor"),
    "large": Config("large", 5_000_000, 3, 32, 1600, 1064, 5, "object360"),
}


def scaled(cfg: Config, P: int | None = None, V: int | None = None, W: int | None = None,
           H: int | None = None, seed: int | None = None, sh_degree: int | None = None) -> Config:
    """A config with some fields overridden (parity tests at oracle-sized shapes)."""
    return Config(cfg.name + "*", P or cfg.P, cfg.sh_degree if sh_degree is None else sh_degree,
                  V or cfg.V, W or cfg.W, H or cfg.H, cfg.seed if seed is None else seed, cfg.layout)


# --------------------------------------------------------------------------- cameras
def look_at(pos, target, W, H, f, znear=0.2):
    """Pinhole camera at `pos` looking at `target`, world +z up, camera +y down."""
    pos = np.asarray(pos, np.float64)
    fwd = np.asarray(target, np.float64) - pos
    fwd /= np.linalg.norm(fwd)
    up = np.array([0.0, 0.0, 1.0])
    right = np.cross(fwd, up)
    if np.linalg.norm(right) < 1e-9:
        right = np.array([1.0, 0.0, 0.0])
    right /= np.linalg.norm(right)
    down = np.cross(fwd, right)
    R = np.stack([right, down, fwd])  # rows: camera axes in world coordinates
    t = -R @ pos
    cam = np.zeros((), CAM_DTYPE)
    cam["R"] = R.reshape(-1).astype(np.float32)
    cam["t"] = t.astype(np.float32)
    cam["fx"] = cam["fy"] = np.float32(f)
    cam["cx"] = np.float32((W - 1) / 2.0)
    cam["cy"] = np.float32((H - 1) / 2.0)
    cam["width"], cam["height"] = W, H
    cam["znear"] = np.float32(znear)
    return cam


def make_camera(R, t, W, H, fx, fy=None, cx=None, cy=None, znear=0.2):
    cam = np.zeros((), CAM_DTYPE)
    cam["R"] = np.asarray(R, np.float32).reshape(-1)
    cam["t"] = np.asarray(t, np.float32)
    cam["fx"] = fx
    cam["fy"] = fx if fy is None else fy
    cam["cx"] = (W - 1) / 2.0 if cx is None else cx
    cam["cy"] = (H - 1) / 2.0 if cy is None else cy
    cam["width"], cam["height"] = W, H
    cam["znear"] = znear
    return cam


def cams_array(cams) -> np.ndarray:
    out = np.zeros(len(cams), CAM_DTYPE)
    for i, c in enumerate(cams):
        out[i] = c
    return out


# --------------------------------------------------------------------------- helpers
def _unit_quats(rng, n):
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    return q


def _quat_from_frame(nrm, rng):
    """Unit quaternion (w,x,y,z) whose rotation maps local z to `nrm`, random twist."""
    n = nrm / np.linalg.norm(nrm, axis=1, keepdims=True)
    a = np.where(np.abs(n[:, :1]) < 0.9, np.array([[1.0, 0, 0]]), np.array([[0, 1.0, 0]]))
    u = np.cross(a, n)
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    v = np.cross(n, u)
    th = rng.uniform(0, 2 * np.pi, size=(len(n), 1))
    u, v = np.cos(th) * u + np.sin(th) * v, -np.sin(th) * u + np.cos(th) * v
    Rm = np.stack([u, v, n], axis=2)  # columns = local axes in world
    # matrix -> quaternion (Shepperd)
    m = Rm
    tr = m[:, 0, 0] + m[:, 1, 1] + m[:, 2, 2]
    q = np.zeros((len(n), 4))
    w = np.sqrt(np.maximum(0, 1 + tr)) / 2
    x = np.sqrt(np.maximum(0, 1 + m[:, 0, 0] - m[:, 1, 1] - m[:, 2, 2])) / 2
    y = np.sqrt(np.maximum(0, 1 - m[:, 0, 0] + m[:, 1, 1] - m[:, 2, 2])) / 2
    z = np.sqrt(np.maximum(0, 1 - m[:, 0, 0] - m[:, 1, 1] + m[:, 2, 2])) / 2
    x = np.copysign(x, m[:, 2, 1] - m[:, 1, 2])
    y = np.copysign(y, m[:, 0, 2] - m[:, 2, 0])
    z = np.copysign(z, m[:, 1, 0] - m[:, 0, 1])
    q[:, 0], q[:, 1], q[:, 2], q[:, 3] = w, x, y, z
    return q / np.linalg.norm(q, axis=1, keepdims=True)


def _finish(rng, means, log_scales, quats, opac_logit, sh_degree, sh0_std=0.6):
    P = len(means)
    K = (sh_degree + 1) ** 2
    sh = np.zeros((P, K, 3), np.float64)
    sh[:, 0, :] = rng.normal(0.0, sh0_std, size=(P, 3))
    for l in range(1, sh_degree + 1):
        sh[:, l * l:(l + 1) * (l + 1), :] = rng.normal(0.0, 0.08 / l, size=(P, 2 * l + 1, 3))
    return dict(
        means=np.ascontiguousarray(means, np.float32),
        log_scales=np.ascontiguousarray(log_scales, np.float32),
        quats=np.ascontiguousarray(quats, np.float32),
        opacity_logits=np.ascontiguousarray(opac_logit, np.float32),
        sh=np.ascontiguousarray(sh, np.float32),
        sh_degree=int(sh_degree),
    )


# --------------------------------------------------------------------------- layouts
def _tiny(cfg: Config, rng):
    """SPEC.md make_synthetic(orbit)."""
    P = cfg.P
    d = rng.normal(size=(P, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    r = rng.uniform(0, 1, size=(P, 1)) ** (1 / 3)
    means = d * r
    scales = rng.uniform(0.01, 0.15, size=(P, 3))
    quats = _unit_quats(rng, P)
    op = rng.uniform(0.3, 0.95, size=P)
    logit = np.log(op / (1 - op))
    rgb = rng.uniform(0, 1, size=(P, 3))
    g = _finish(rng, means, np.log(scales), quats, logit, cfg.sh_degree)
    g["sh"][:, 0, :] = ((rgb - 0.5) / SH_C0).astype(np.float32)
    cams = []
    for k in range(cfg.V):
        a = 2 * np.pi * k / cfg.V
        cams.append(look_at([3 * np.cos(a), 3 * np.sin(a), 0.0], [0, 0, 0], cfg.W, cfg.H, 0.9 * cfg.W))
    return g, cams_array(cams)


def _object360(cfg: Config, rng, stretch_x=1.0):
    P = cfg.P
    n_surf = int(round(0.75 * P))
    n_vol = P - n_surf
    w = np.array([0.40, 0.35, 0.25])
    counts = np.floor(w * n_surf).astype(int)
    counts[0] += n_surf - counts.sum()
    pts, nrm, s0s = [], [], []
    # ground disc z=0, r<=4
    n = counts[0]
    rr = 4 * np.sqrt(rng.uniform(0, 1, n))
    th = rng.uniform(0, 2 * np.pi, n)
    pts.append(np.stack([rr * np.cos(th), rr * np.sin(th), np.zeros(n)], 1))
    nrm.append(np.tile([0.0, 0.0, 1.0], (n, 1)))
    s0s.append(np.full(n, 1.2 * math.sqrt(math.pi * 16 / max(n, 1))))
    # ellipsoid shell radii (1,1,0.6) centred (0,0,0.6)
    n = counts[1]
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    rad = np.array([1.0, 1.0, 0.6])
    pts.append(d * rad + np.array([0, 0, 0.6]))
    nn = d / rad
    nrm.append(nn / np.linalg.norm(nn, axis=1, keepdims=True))
    s0s.append(np.full(n, 1.2 * math.sqrt(9.8 / max(n, 1))))
    # background cylinder r=6, z in [0,4]
    n = counts[2]
    th = rng.uniform(0, 2 * np.pi, n)
    z = rng.uniform(0, 4, n)
    pts.append(np.stack([6 * np.cos(th), 6 * np.sin(th), z], 1))
    nrm.append(np.stack([-np.cos(th), -np.sin(th), np.zeros(n)], 1))
    s0s.append(np.full(n, 1.2 * math.sqrt(2 * math.pi * 6 * 4 / max(n, 1))))
    pts = np.concatenate(pts)
    nrm = np.concatenate(nrm)
    s0 = np.concatenate(s0s)
    pts = pts + rng.normal(0, 0.01, size=pts.shape)
    ls = np.log(s0)[:, None] + rng.normal(0, 0.4, size=(n_surf, 3))
    ls[:, 2] += math.log(0.15)  # flat along the surface normal (local z)
    q = _quat_from_frame(nrm, rng)
    # volume Gaussians uniform in the cylinder
    rr = 6 * np.sqrt(rng.uniform(0, 1, n_vol))
    th = rng.uniform(0, 2 * np.pi, n_vol)
    vpts = np.stack([rr * np.cos(th), rr * np.sin(th), rng.uniform(0, 4, n_vol)], 1)
    s_vol = 1.5 * 1.2 * math.sqrt(2 * math.pi * 6 * 4 / max(counts[2], 1))
    # near-isotropic (N(0, 0.1²) log-scale jitter): an exactly isotropic Gaussian has an
    # identically-zero rotation gradient, a degenerate case tested on its own
    vls = math.log(s_vol) + rng.normal(0, 0.1, size=(n_vol, 3))
    vq = _unit_quats(rng, n_vol)
    means = np.concatenate([pts, vpts])
    means[:, 0] *= stretch_x
    log_scales = np.concatenate([ls, vls])
    quats = np.concatenate([q, vq])
    perm = rng.permutation(P)  # interleave surface/volume so gid carries no structure
    means, log_scales, quats = means[perm], log_scales[perm], quats[perm]
    hi = rng.uniform(0, 1, P) < 0.6
    logit = np.where(hi, rng.normal(3, 1, P), rng.normal(-2, 1.5, P))
    g = _finish(rng, means, log_scales, quats, logit, cfg.sh_degree)
    cams = []
    for k in range(cfg.V):
        yaw = 2 * np.pi * k / cfg.V + np.deg2rad(rng.uniform(-5, 5))
        h = 1.0 + rng.uniform(-0.3, 0.3)
        pos = [3.2 * stretch_x * np.cos(yaw), 3.2 * np.sin(yaw), h]
        cams.append(look_at(pos, [0, 0, 0.5], cfg.W, cfg.H, 0.9 * cfg.W))
    return g, cams_array(cams)


def _indoor(cfg: Config, rng):
    P = cfg.P
    n_wall = int(round(0.7 * P))
    n_box = P - n_wall
    L = np.array([6.0, 8.0, 3.0])  # room [-3,3]x[-4,4]x[0,3]
    lo = np.array([-3.0, -4.0, 0.0])
    areas = np.array([L[1] * L[2], L[1] * L[2], L[0] * L[2], L[0] * L[2], L[0] * L[1], L[0] * L[1]])
    face = rng.choice(6, size=n_wall, p=areas / areas.sum())
    u = rng.uniform(0, 1, size=(n_wall, 3))
    pts = lo + u * L
    ax = face // 2
    side = face % 2
    pts[np.arange(n_wall), ax] = lo[ax] + side * L[ax]
    nrm = np.zeros((n_wall, 3))
    nrm[np.arange(n_wall), ax] = np.where(side == 0, 1.0, -1.0)
    s0w = 1.2 * math.sqrt(areas.sum() / max(n_wall, 1))
    # 12 random inner boxes
    bc = rng.uniform(lo + 0.8, lo + L - 0.8, size=(12, 3))
    bc[:, 2] = rng.uniform(0.3, 1.0, 12)
    bs = rng.uniform(0.2, 0.6, size=(12, 3))
    bi = rng.integers(0, 12, n_box)
    f = rng.integers(0, 6, n_box)
    bu = rng.uniform(-1, 1, size=(n_box, 3))
    bax = f // 2
    bu[np.arange(n_box), bax] = np.where(f % 2 == 0, -1.0, 1.0)
    bpts = bc[bi] + bu * bs[bi]
    bn = np.zeros((n_box, 3))
    bn[np.arange(n_box), bax] = np.where(f % 2 == 0, -1.0, 1.0)
    box_area = (8 * (bs[:, 0] * bs[:, 1] + bs[:, 1] * bs[:, 2] + bs[:, 0] * bs[:, 2])).sum()
    s0b = 1.2 * math.sqrt(box_area / max(n_box, 1))
    pts = np.concatenate([pts, bpts]) + rng.normal(0, 0.01, size=(P, 3))
    nrm = np.concatenate([nrm, bn])
    s0 = np.concatenate([np.full(n_wall, s0w), np.full(n_box, s0b)])
    ls = np.log(s0)[:, None] + rng.normal(0, 0.4, size=(P, 3))
    ls[:, 2] += math.log(0.15)
    q = _quat_from_frame(nrm, rng)
    perm = rng.permutation(P)
    pts, ls, q = pts[perm], ls[perm], q[perm]
    hi = rng.uniform(0, 1, P) < 0.6
    logit = np.where(hi, rng.normal(3, 1, P), rng.normal(-2, 1.5, P))
    g = _finish(rng, pts, ls, q, logit, cfg.sh_degree)
    cams = []
    for k in range(cfg.V):
        pos = np.array([rng.uniform(-1.5, 1.5), rng.uniform(-2, 2), 1.5])
        yaw = rng.uniform(0, 2 * np.pi)
        tgt = pos + np.array([np.cos(yaw), np.sin(yaw), rng.uniform(-0.2, 0.1)])
        cams.append(look_at(pos, tgt, cfg.W, cfg.H, 0.8 * cfg.W))
    return g, cams_array(cams)


def make_scene(cfg: Config | str, seed: int | None = None):
    """Return (gaussians: dict of float32 arrays + sh_degree, cams: CAM_DTYPE[V])."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    rng = np.random.Generator(np.random.PCG64(cfg.seed if seed is None else seed))
    if cfg.layout == "tiny":
        return _tiny(cfg, rng)
    if cfg.layout == "object360":
        return _object360(cfg, rng)
    if cfg.layout == "object360x":
        return _object360(cfg, rng, stretch_x=2.5)
    if cfg.layout == "indoor":
        return _indoor(cfg, rng)
    raise ValueError(cfg.layout)


def make_dLdC(V: int, H: int, W: int, seed: int) -> np.ndarray:
    """Per-pixel ∂L/∂C of an ℓ1 photometric loss against an unknown target:
    sign(C − C*)/(3·V·H·W) with the signs drawn at random. float32 [V,3,H,W]."""
    rng = np.random.Generator(np.random.PCG64(seed + 100))
    s = rng.integers(0, 2, size=(V, 3, H, W)).astype(np.float32) * 2.0 - 1.0
    return (s / np.float32(3 * V * H * W)).astype(np.float32)


def make_dLdC_scaled(V: int, H: int, W: int, seed: int) -> np.ndarray:
    """Same sign pattern with O(1) magnitude (used by small parity cases so that
    fp32 rounding is compared at a sensible scale)."""
    return make_dLdC(V, H, W, seed) * np.float32(3 * V * H * W)


def subset_views(cams: np.ndarray, lo: int, hi: int) -> np.ndarray:
    return np.ascontiguousarray(cams[lo:hi])


def make_dssim_inputs(V: int, H: int, W: int, seed: int, bg_frac: float = 0.15):
    """Seeded inputs for the NEXT-2 D-SSIM (DESIGN.md §14 recipe): a rendered-like
    image (smooth colour ramps + texture, in [0, 1]), a target = image + noise,
    a depth map of two slanted planes with a step edge between them (2–7 units,
    the object360 depth range) and a background region (T_final = 1, depth 0)
    in a corner disc; foreground T_final ∈ [0, 0.3].  Returns float32 arrays
    img, target [V,3,H,W], depth, T_final [V,H,W] and a cams array (f = 0.9·W)."""
    rng = np.random.Generator(np.random.PCG64(seed + 500))
    y, x = np.mgrid[0:H, 0:W].astype(np.float64)
    img = np.empty((V, 3, H, W))
    depth = np.empty((V, H, W))
    Tf = np.empty((V, H, W))
    cams = []
    for v in range(V):
        for c in range(3):
            a, b, ph = rng.uniform(-1, 1, 3)
            img[v, c] = 0.5 + 0.25 * (a * x / W + b * y / H) + 0.15 * np.sin(ph * 6 + x * 0.7 + y * 0.3 * (c + 1))
        img[v] += rng.normal(0, 0.05, (3, H, W))
        edge = rng.uniform(0.35, 0.65) * W
        near = 2.0 + rng.uniform(0, 1) + 0.01 * (x - W / 2) + 0.005 * y
        far = 5.0 + rng.uniform(0, 1) - 0.008 * y
        depth[v] = np.where(x < edge + 0.2 * (y - H / 2), near, far)
        r = np.hypot(x - W, y - H)
        bgm = r < np.sqrt(bg_frac * 4 * W * H / np.pi)
        Tf[v] = rng.uniform(0.0, 0.3, (H, W))
        Tf[v][bgm] = 1.0
        depth[v][bgm] = 0.0
        cams.append(make_camera(np.eye(3), [0, 0, 0], W, H, 0.9 * W))
    img = np.clip(img, 0, 1)
    tgt = np.clip(img + rng.normal(0, 0.08, img.shape), 0, 1)
    return (img.astype(np.float32), tgt.astype(np.float32), depth.astype(np.float32), Tf.astype(np.float32),
            cams_array(cams))


def make_adc_inputs(P: int, seed: int, N: int = 2, sh_degree: int = 3, iters: int = 100, B: int = 4):
    """Seeded inputs for the NEXT-3 ADC step (DESIGN.md §15 recipe): Gaussians from the
    object360 generator's distributions (log-scales around ln 0.005, about half "large" at 0.01, opacities U[0.002, 0.95]),
    running accumulators of `iters` steps of B views — denom ~ integer U[0, B·iters] with 10%
    never visible, per-visibility mean E1 log-normal around 1e-4 (≈16% above the 3DGS 2e-4), E2 = E1·U[0.3, 1],
    E_old = E2·U[0, 1] (the triangle-inequality order E1 ≥ E2 ≥ E_old) — and the split noise
    n ~ N(0, I) [P, N, 3]."""
    rng = np.random.Generator(np.random.PCG64(seed + 900))
    means = rng.normal(0, 1.0, (P, 3))
    log_scales = np.log(0.005) + rng.normal(0, 0.8, (P, 3))
    quats = _unit_quats(rng, P)
    op = rng.uniform(0.002, 0.95, P)
    g = _finish(rng, means, log_scales, quats, np.log(op / (1 - op)), sh_degree)
    den = rng.integers(0, B * iters + 1, P).astype(np.float32)
    den[rng.uniform(0, 1, P) < 0.1] = 0
    e1 = (den * np.exp(rng.normal(np.log(1e-4), 0.7, P))).astype(np.float32)
    e2 = (e1 * rng.uniform(0.3, 1.0, P)).astype(np.float32)
    eo = (e2 * rng.uniform(0.0, 1.0, P)).astype(np.float32)
    acc = dict(e1=e1, e2=e2, e_old=eo, denom=den)
    noise = rng.normal(0, 1, (P, N, 3)).astype(np.float32)
    return g, acc, noise


def make_lab_targets(V: int, H: int, W: int, seed: int) -> np.ndarray:
    """Seeded target photos for the NEXT-4 variance lab: per view a smooth
    colour field (random linear ramps + low-frequency sinusoids) in [0, 1], float32 [V,3,H,W].
    Independent of any scene: the lab only needs a fixed per-view loss landscape."""
    rng = np.random.Generator(np.random.PCG64(seed + 1300))
    y, x = np.mgrid[0:H, 0:W].astype(np.float64)
    out = np.empty((V, 3, H, W))
    for v in range(V):
        for c in range(3):
            a, b, f1, f2, ph = rng.uniform(-1, 1, 5)
            out[v, c] = 0.4 + 0.2 * (a * x / W + b * y / H) + 0.2 * np.sin(2 * np.pi * (f1 * x / W + f2 * y / H) + 3 * ph)
    return np.clip(out, 0, 1).astype(np.float32)
