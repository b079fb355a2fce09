"""Thin ctypes binding of libmvgs.so (include/mvgs.h).  Argument marshalling
only: every step of the path runs in the library's sm_100a kernels.  PyTorch
provides device memory and the stream handle.  There is no fallback — if the
library is missing or fails to load, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MVGS_LIB", os.path.join(HERE, "libmvgs.so"))  # override: experiments only

MVGS_OK, MVGS_ERR_INVALID, MVGS_ERR_CAPACITY, MVGS_ERR_STATE, MVGS_ERR_CUDA = 0, -1, -2, -3, -4
NG = 10
PG_STRIDE = 12  # floats per per-pair gradient slot

# the exported symbols include/mvgs.h declares (checked by tests/test_abi.py)
SYMBOLS = ["mvgs_create", "mvgs_destroy", "mvgs_last_error", "mvgs_reserve", "mvgs_preprocess", "mvgs_render_fwd",
           "mvgs_render_bwd", "mvgs_adc_stats", "mvgs_adc_stats_range", "mvgs_query", "mvgs_export_lists", "mvgs_export_pairs",
           "mvgs_set_timing", "mvgs_stage_times", "mvgs_set_eval_counting", "mvgs_render_fwd_partial", "mvgs_render_bwd_partial",
           "mvgs_render_fwd_depth", "mvgs_dssim3d", "mvgs_adc_step", "mvgs_adc_remap",
           "mvgs_loss_grad", "mvgs_loss_grad_u8", "mvgs_render_bwd_l1", "mvgs_grad_moments", "mvgs_grad_variance", "mvgs_set_debug_blend_counts", "mvgs_set_tma",
           "mvgs_owner_slices", "mvgs_owner_prepare", "mvgs_owner_adc_stats", "mvgs_e_old_from_gsum"]
PARTIAL_THREAD_EFFICIENT, PARTIAL_MASKED = 0, 1
STAGE_NAMES = ["count", "scan_pairs", "project", "scan_buckets", "sort_pairs", "dup", "sort_entries", "render_fwd",
               "render_bwd", "gauss_bwd", "dssim"]


class MvgsError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"mvgs status {status}: {msg}")
        self.status = status


class Gaussians(C.Structure):
    _fields_ = [("P", C.c_int64), ("sh_degree", C.c_int32), ("sh_stride", C.c_int32), ("means", C.c_void_p),
                ("log_scales", C.c_void_p), ("quats", C.c_void_p), ("opacity_logits", C.c_void_p),
                ("sh", C.c_void_p)]


class Grads(C.Structure):
    _fields_ = [(k, C.c_void_p) for k in ("d_means", "d_log_scales", "d_quats", "d_opacity_logits", "d_sh")]


ADC_FIELDS = ("e1", "e2", "e_old", "vis", "e1_acc", "e2_acc", "denom_acc", "e_old_acc", "max_radius", "gsum")


class Adc(C.Structure):
    _fields_ = [(k, C.c_void_p) for k in ADC_FIELDS]


class AdcConfig(C.Structure):
    _fields_ = [("grad_threshold_split", C.c_float), ("grad_threshold_clone", C.c_float),
                ("size_threshold", C.c_float), ("split_factor", C.c_float), ("split_count", C.c_int32),
                ("prune_opacity", C.c_float), ("prune_scale_max", C.c_float), ("metric_mode", C.c_int32),
                ("batch_views", C.c_int32)]


class AdcAccum(C.Structure):
    _fields_ = [(k, C.c_void_p) for k in ("e1_acc", "e2_acc", "e_old_acc", "denom_acc")]


class GaussiansOut(C.Structure):
    _fields_ = [("capacity", C.c_int64), ("sh_stride", C.c_int32), ("means", C.c_void_p), ("log_scales", C.c_void_p),
                ("quats", C.c_void_p), ("opacity_logits", C.c_void_p), ("sh", C.c_void_p)]


class AdcReport(C.Structure):
    _fields_ = [(k, C.c_int64) for k in ("n_split", "n_clone", "n_pruned", "P_new")]


class Stats(C.Structure):
    _fields_ = [("Q", C.c_int64), ("K", C.c_int64), ("cap_pairs", C.c_int64), ("cap_entries", C.c_int64),
                ("max_bucket", C.c_int64), ("n_visible", C.c_int64), ("overflow", C.c_int32), ("V", C.c_int32),
                ("tiles_x", C.c_int32), ("tiles_y", C.c_int32), ("eval_fwd", C.c_int64), ("eval_bwd", C.c_int64),
                ("exp_fwd", C.c_int64), ("exp_bwd", C.c_int64), ("threads_launched", C.c_int64),
                ("threads_active", C.c_int64), ("lane_steps_launched", C.c_int64), ("lane_steps_active", C.c_int64)]


CAM_BYTES = 76


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(LIB_PATH)
    vp, st, i64 = C.c_void_p, C.c_int, C.c_int64
    L.mvgs_create.argtypes = [C.POINTER(vp), C.c_int, i64, i64]
    L.mvgs_destroy.argtypes = [vp]
    L.mvgs_destroy.restype = None
    L.mvgs_last_error.argtypes = [vp]
    L.mvgs_last_error.restype = C.c_char_p
    L.mvgs_reserve.argtypes = [vp, i64, i64]
    L.mvgs_preprocess.argtypes = [vp, C.POINTER(Gaussians), vp, C.c_int32, vp, vp]
    L.mvgs_render_fwd.argtypes = [vp, vp, vp, vp, vp]
    L.mvgs_render_fwd_depth.argtypes = [vp, vp, vp, vp, vp, vp]
    L.mvgs_render_bwd.argtypes = [vp, vp, vp, vp, vp]
    L.mvgs_adc_stats.argtypes = [vp, C.POINTER(Grads), C.POINTER(Adc), vp]
    L.mvgs_adc_stats_range.argtypes = [vp, C.c_int64, C.c_int64, C.POINTER(Grads), C.POINTER(Adc), vp]
    L.mvgs_query.argtypes = [vp, C.POINTER(Stats)]
    L.mvgs_export_lists.argtypes = [vp, vp, vp, vp]
    L.mvgs_export_pairs.argtypes = [vp, vp, vp, vp, vp, vp]
    L.mvgs_set_timing.argtypes = [vp, C.c_int]
    L.mvgs_set_eval_counting.argtypes = [vp, C.c_int]
    L.mvgs_set_tma.argtypes = [vp, C.c_int]
    L.mvgs_owner_slices.argtypes = [vp, vp, C.c_int32, vp, vp, vp]
    L.mvgs_owner_prepare.argtypes = [vp, vp, C.c_int32, C.c_int64, C.c_int64, vp, vp, vp]
    L.mvgs_owner_adc_stats.argtypes = [vp, vp, vp, vp]
    L.mvgs_e_old_from_gsum.argtypes = [vp, vp, C.c_int64, vp, vp, vp]
    L.mvgs_set_debug_blend_counts.argtypes = [vp, vp]
    L.mvgs_render_fwd_partial.argtypes = [vp, vp, C.c_int32, C.c_int32, vp, vp, vp, vp]
    L.mvgs_render_bwd_partial.argtypes = [vp, vp, C.c_int32, C.c_int32, vp, vp, vp, vp]
    L.mvgs_dssim3d.argtypes = [vp, vp, C.c_int32, C.c_int32, C.c_int32, vp, vp, vp, vp, C.c_float, vp, vp, vp]
    L.mvgs_adc_step.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]
    L.mvgs_adc_remap.argtypes = [vp, vp, vp, i64, vp, vp, i64, vp]
    L.mvgs_loss_grad.argtypes = [vp, vp, vp, i64, C.c_int32, C.c_float, vp, vp, vp]
    L.mvgs_loss_grad_u8.argtypes = [vp, vp, vp, i64, C.c_int32, C.c_float, vp, vp, vp]
    L.mvgs_render_bwd_l1.argtypes = [vp, vp, vp, C.c_float, vp, vp, vp, vp]
    L.mvgs_grad_moments.argtypes = [vp, vp, i64, vp, vp, vp]
    L.mvgs_grad_variance.argtypes = [vp, vp, i64, vp, i64, vp, vp]
    L.mvgs_stage_times.argtypes = [vp, C.POINTER(C.c_float), C.c_int]
    L.mvgs_stage_times.restype = C.c_int
    for n in SYMBOLS:
        if n not in ("mvgs_destroy", "mvgs_last_error", "mvgs_stage_times"):
            getattr(L, n).restype = st
    return L


_lib = _load()


def lib():
    return _lib


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, torch.Tensor):
        if not t.is_cuda or not t.is_contiguous():
            raise ValueError("mvgs: tensors must be contiguous CUDA tensors")
        return t.data_ptr()
    return t


def _stream(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


def _check(ctx, status):
    if status != MVGS_OK:
        msg = _lib.mvgs_last_error(ctx).decode() if ctx else ""
        raise MvgsError(status, msg)


def create(device: int = 0, max_pairs: int = 0, max_entries: int = 0):
    h = C.c_void_p()
    _check(None, _lib.mvgs_create(C.byref(h), device, max_pairs, max_entries))
    return h


def destroy(ctx):
    if ctx:
        _lib.mvgs_destroy(ctx)


def reserve(ctx, max_pairs: int, max_entries: int):
    _check(ctx, _lib.mvgs_reserve(ctx, int(max_pairs), int(max_entries)))


def gaussians_struct(g: dict) -> Gaussians:
    sh = g["sh"]
    return Gaussians(int(g["means"].shape[0]), int(g["sh_degree"]), int(sh.shape[1]), _ptr(g["means"]),
                     _ptr(g["log_scales"]), _ptr(g["quats"]), _ptr(g["opacity_logits"]), _ptr(sh))


def preprocess(ctx, g: dict, cams: np.ndarray, bg=(0.0, 0.0, 0.0), stream=None):
    """S1–S5.  `g`: dict of contiguous fp32 CUDA tensors (+ int sh_degree);
    `cams`: numpy structured array with the 76-byte mvgs_camera layout."""
    cams = np.ascontiguousarray(cams)
    assert cams.dtype.itemsize == CAM_BYTES
    bgh = np.ascontiguousarray(bg, np.float32)
    gs = gaussians_struct(g)
    _check(ctx, _lib.mvgs_preprocess(ctx, C.byref(gs), cams.ctypes.data, len(cams), bgh.ctypes.data, _stream(stream)))


def render_fwd(ctx, rgb, T_final, n_contrib, stream=None):
    _check(ctx, _lib.mvgs_render_fwd(ctx, _ptr(rgb), _ptr(T_final), _ptr(n_contrib), _stream(stream)))


def render_fwd_depth(ctx, rgb, T_final, n_contrib, depth, stream=None):
    _check(ctx, _lib.mvgs_render_fwd_depth(ctx, _ptr(rgb), _ptr(T_final), _ptr(n_contrib), _ptr(depth),
                                           _stream(stream)))


def dssim3d(ctx, cams: np.ndarray, img, target, depth, T_final, loss, dL_dimg=None, sigma_px: float = 1.5,
            stream=None):
    """NEXT-2: 3D distance-aware D-SSIM.  img/target [V,3,H,W],
    depth/T_final [V,H,W], loss [1] (device fp32); dL_dimg [V,3,H,W] or None."""
    cams = np.ascontiguousarray(cams)
    assert cams.dtype.itemsize == CAM_BYTES
    V, _, H, W = img.shape
    _check(ctx, _lib.mvgs_dssim3d(ctx, cams.ctypes.data, V, H, W, _ptr(img), _ptr(target), _ptr(depth), _ptr(T_final),
                                  float(sigma_px), _ptr(loss), _ptr(dL_dimg), _stream(stream)))


def render_bwd(ctx, dL_drgb, T_final, n_contrib, stream=None):
    _check(ctx, _lib.mvgs_render_bwd(ctx, _ptr(dL_drgb), _ptr(T_final), _ptr(n_contrib), _stream(stream)))


def render_bwd_l1(ctx, rgb, target_u8, T_final, n_contrib, scale: float | None = None, loss=None, stream=None):
    """S7 with the ℓ1 loss of 8-bit targets fused in (∂L/∂C formed in the kernel; mean by default)."""
    sc = 1.0 / int(rgb.numel()) if scale is None else scale
    _check(ctx, _lib.mvgs_render_bwd_l1(ctx, _ptr(rgb), _ptr(target_u8), float(sc), _ptr(T_final), _ptr(n_contrib),
                                        _ptr(loss), _stream(stream)))


def render_fwd_partial(ctx, pix, S: int, mode: int, rgb, T_final, n_contrib, stream=None):
    """NEXT-1 (Alg. 3): render only the listed pixels (pix [V,T,S] int32, local 0..255)."""
    _check(ctx, _lib.mvgs_render_fwd_partial(ctx, _ptr(pix), int(S), int(mode), _ptr(rgb), _ptr(T_final),
                                             _ptr(n_contrib), _stream(stream)))


def render_bwd_partial(ctx, pix, S: int, mode: int, dL_drgb, T_final, n_contrib, stream=None):
    _check(ctx, _lib.mvgs_render_bwd_partial(ctx, _ptr(pix), int(S), int(mode), _ptr(dL_drgb), _ptr(T_final),
                                             _ptr(n_contrib), _stream(stream)))


def adc_stats(ctx, grads: dict, adc: dict, stream=None):
    gr = Grads(*[_ptr(grads[k]) for k in ("d_means", "d_log_scales", "d_quats", "d_opacity_logits", "d_sh")])
    ad = Adc(*[_ptr(adc.get(k)) for k in ADC_FIELDS])
    _check(ctx, _lib.mvgs_adc_stats(ctx, C.byref(gr), C.byref(ad), _stream(stream)))


def adc_stats_range(ctx, g_begin: int, g_end: int, grads: dict, adc: dict, stream=None):
    """S8–S9 for Gaussians [g_begin, g_end) (g_begin % 256 == 0); the tensors hold rows g_begin.. ."""
    gr = Grads(*[_ptr(grads[k]) for k in ("d_means", "d_log_scales", "d_quats", "d_opacity_logits", "d_sh")])
    ad = Adc(*[_ptr(adc.get(k)) for k in ADC_FIELDS])
    _check(ctx, _lib.mvgs_adc_stats_range(ctx, int(g_begin), int(g_end), C.byref(gr), C.byref(ad), _stream(stream)))


ADC_DEFAULTS = dict(grad_threshold_split=2e-4, grad_threshold_clone=2e-4, size_threshold=0.01, split_factor=1.6,
                    split_count=2, prune_opacity=0.005, prune_scale_max=0.0, metric_mode=1, batch_views=1)


def alloc_gaussians(capacity: int, sh_stride: int, device) -> dict:
    f = dict(dtype=torch.float32, device=device)
    return dict(means=torch.empty((capacity, 3), **f), log_scales=torch.empty((capacity, 3), **f),
                quats=torch.empty((capacity, 4), **f), opacity_logits=torch.empty((capacity,), **f),
                sh=torch.empty((capacity, sh_stride, 3), **f))


def adc_step(ctx, g: dict, acc: dict, noise, cfg: dict, out: dict, origin, kind, stream=None) -> dict:
    """NEXT-3 (P:4): one ADC event.  `acc` holds e1_acc / e2_acc / e_old_acc /
    denom_acc device tensors, `noise` [P, N, 3] standard normals, `out` arrays from
    alloc_gaussians(capacity, ...).  Returns the report; raises MvgsError (status −2) when the
    new count exceeds the capacity (the report is attached as .report)."""
    c = dict(ADC_DEFAULTS)
    c.update(cfg)
    conf = AdcConfig(**c)
    gs = gaussians_struct(g)
    ac = AdcAccum(*[_ptr(acc.get(k)) for k in ("e1_acc", "e2_acc", "e_old_acc", "denom_acc")])
    o = GaussiansOut(int(out["means"].shape[0]), int(out["sh"].shape[1]), _ptr(out["means"]), _ptr(out["log_scales"]),
                     _ptr(out["quats"]), _ptr(out["opacity_logits"]), _ptr(out["sh"]))
    rep = AdcReport()
    st = _lib.mvgs_adc_step(ctx, C.byref(gs), C.byref(ac), _ptr(noise), C.byref(conf), C.byref(o), _ptr(origin),
                            _ptr(kind), C.byref(rep), _stream(stream))
    r = {k: getattr(rep, k) for k, _ in AdcReport._fields_}
    if st != MVGS_OK:
        e = MvgsError(st, _lib.mvgs_last_error(ctx).decode())
        e.report = r
        raise e
    return r


def adc_remap(ctx, src, dst, origin, kind, P_new: int, stream=None):
    width = int(src[0].numel()) if src.dim() > 1 else 1
    _check(ctx, _lib.mvgs_adc_remap(ctx, _ptr(src), _ptr(dst), width, _ptr(origin), _ptr(kind), int(P_new),
                                    _stream(stream)))


LOSS_L1, LOSS_L2 = 0, 1


def loss_grad(ctx, rgb, target, dL, mode: int = LOSS_L1, scale: float | None = None, loss=None, stream=None):
    """NEXT-4: ∂loss/∂C of a rendered batch (ℓ1 or ℓ2, mean over all elements by default)."""
    n = int(rgb.numel())
    sc = 1.0 / n if scale is None else scale
    fn = _lib.mvgs_loss_grad_u8 if target.dtype == torch.uint8 else _lib.mvgs_loss_grad  # 8-bit images: t/255
    _check(ctx, fn(ctx, _ptr(rgb), _ptr(target), n, int(mode), float(sc), _ptr(dL), _ptr(loss), _stream(stream)))


def grad_moments(ctx, g, acc_sum, acc_sumsq, stream=None):
    """NEXT-4: acc_sum (fp64 [n]) += g, acc_sumsq (fp64 [1]) += ‖g‖²."""
    _check(ctx, _lib.mvgs_grad_moments(ctx, _ptr(g), int(g.numel()), _ptr(acc_sum), _ptr(acc_sumsq), _stream(stream)))


def grad_variance(ctx, acc_sum, acc_sumsq, K: int, out, stream=None):
    """NEXT-4: 𝕍 = (1/K)Σ‖g_k‖² − ‖(1/K)Σ g_k‖² into out (fp64 [1])."""
    _check(ctx, _lib.mvgs_grad_variance(ctx, _ptr(acc_sum), int(acc_sum.numel()), _ptr(acc_sumsq), int(K), _ptr(out),
                                        _stream(stream)))


def query(ctx, raise_on_capacity: bool = True) -> dict:
    s = Stats()
    st = _lib.mvgs_query(ctx, C.byref(s))
    if st != MVGS_OK and not (st == MVGS_ERR_CAPACITY and not raise_on_capacity):
        _check(ctx, st)
    return {k: getattr(s, k) for k, _ in Stats._fields_}


def export_lists(ctx, range_start, entry_gid, stream=None):
    _check(ctx, _lib.mvgs_export_lists(ctx, _ptr(range_start), _ptr(entry_gid), _stream(stream)))


def export_pairs(ctx, pair_ids=None, pair_i=None, pair_f=None, pair_g=None, stream=None):
    _check(ctx, _lib.mvgs_export_pairs(ctx, _ptr(pair_ids), _ptr(pair_i), _ptr(pair_f), _ptr(pair_g),
                                       _stream(stream)))


def set_debug_blend_counts(ctx, nblend=None):
    """Parity export: per-pixel count of entries the backward blended ([V,H,W] int32), or off."""
    _check(ctx, _lib.mvgs_set_debug_blend_counts(ctx, _ptr(nblend) if nblend is not None else None))


def set_timing(ctx, enable: bool):
    _check(ctx, _lib.mvgs_set_timing(ctx, int(bool(enable))))


class DeviceArray:
    """Zero-copy view of context-owned device memory (float32) for torch (cuda array interface)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": "<f4", "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def _as_tensor(ptr: int, n: int):
    return torch.as_tensor(DeviceArray(ptr, n), device="cuda") if n > 0 else torch.empty(0, device="cuda")


def owner_slices(ctx, g_bounds, V: int, stream=None):
    """(slot_off [V, N+1] int64, slot tensor [Q·12] float32 view of the context's gradient slots)."""
    gb = np.ascontiguousarray(g_bounds, np.int64)
    N = len(gb) - 1
    off = np.zeros((V, N + 1), np.int64)
    p = C.c_void_p()
    _check(ctx, _lib.mvgs_owner_slices(ctx, gb.ctypes.data, N, off.ctypes.data, C.byref(p), _stream(stream)))
    return off, _as_tensor(p.value, int(off[-1, -1]) * PG_STRIDE if V else 0)


def owner_prepare(ctx, cams_all, g_begin: int, g_end: int, stream=None):
    """(view_off [V_all+1] int64, receive tensor [view_off[-1]·12] float32, context-owned)."""
    cams_all = np.ascontiguousarray(cams_all)
    V = len(cams_all)
    off = np.zeros(V + 1, np.int64)
    p = C.c_void_p()
    _check(ctx, _lib.mvgs_owner_prepare(ctx, cams_all.ctypes.data, V, int(g_begin), int(g_end), off.ctypes.data,
                                        C.byref(p), _stream(stream)))
    return off, _as_tensor(p.value, int(off[-1]) * PG_STRIDE)


def owner_adc_stats(ctx, grads: dict, adc: dict, stream=None):
    gr = Grads(*[_ptr(grads[k]) for k in ("d_means", "d_log_scales", "d_quats", "d_opacity_logits", "d_sh")])
    ad = Adc(*[_ptr(adc.get(k)) for k in ADC_FIELDS])
    _check(ctx, _lib.mvgs_owner_adc_stats(ctx, C.byref(gr), C.byref(ad), _stream(stream)))


def e_old_from_gsum(ctx, gsum, e_old=None, e_old_acc=None, stream=None):
    """E_old = ‖gsum‖ per Gaussian (gsum [n,2] device fp32), into e_old and/or += e_old_acc."""
    n = int(gsum.shape[0])
    _check(ctx, _lib.mvgs_e_old_from_gsum(ctx, _ptr(gsum), n, _ptr(e_old), _ptr(e_old_acc), _stream(stream)))


def set_tma(ctx, enable: bool):
    """Forward staging by TMA gather4 (bit-identical results; off by default, measured slower)."""
    _check(ctx, _lib.mvgs_set_tma(ctx, int(bool(enable))))


def set_eval_counting(ctx, enable: bool):
    _check(ctx, _lib.mvgs_set_eval_counting(ctx, int(bool(enable))))


def stage_times(ctx) -> dict:
    """Milliseconds of the most recent run of each stage (synchronises)."""
    buf = (C.c_float * len(STAGE_NAMES))()
    n = _lib.mvgs_stage_times(ctx, buf, len(STAGE_NAMES))
    return {STAGE_NAMES[i]: float(buf[i]) for i in range(n)}


class Rasterizer:
    """Convenience owner of one context: sizes capacities, allocates outputs and
    runs preprocess → render_fwd → render_bwd → adc_stats.  Marshalling only."""

    def __init__(self, device: int = 0, max_pairs: int = 0, max_entries: int = 0):
        self.device = device
        self.ctx = create(device, max_pairs, max_entries)
        self.V = self.H = self.W = 0

    def __del__(self):
        ctx = getattr(self, "ctx", None)
        if ctx:
            destroy(ctx)
            self.ctx = None

    def preprocess(self, g: dict, cams: np.ndarray, bg=(0.0, 0.0, 0.0), stream=None, auto_reserve: bool = True):
        self.g = g
        self.cams = np.ascontiguousarray(cams)
        self.bg = bg
        self.V = len(cams)
        self.W = int(cams[0]["width"])
        self.H = int(cams[0]["height"])
        preprocess(self.ctx, g, self.cams, bg, stream)
        if auto_reserve:
            st = query(self.ctx, raise_on_capacity=False)
            for _ in range(3):
                if not st["overflow"]:
                    break
                reserve(self.ctx, int(st["Q"] * 1.1) + 1024, int(st["K"] * 1.1) + 4096)
                preprocess(self.ctx, g, self.cams, bg, stream)
                st = query(self.ctx, raise_on_capacity=False)
            if st["overflow"]:
                query(self.ctx)  # raises with the library's message
            self.stats = st

    def alloc_forward(self):
        dev = torch.device("cuda", self.device)
        rgb = torch.empty((self.V, 3, self.H, self.W), dtype=torch.float32, device=dev)
        Tf = torch.empty((self.V, self.H, self.W), dtype=torch.float32, device=dev)
        nc = torch.empty((self.V, self.H, self.W), dtype=torch.int32, device=dev)
        return rgb, Tf, nc

    def forward(self, out=None, stream=None):
        rgb, Tf, nc = out if out is not None else self.alloc_forward()
        render_fwd(self.ctx, rgb, Tf, nc, stream)
        self._fwd = (Tf, nc)
        return rgb, Tf, nc

    def alloc_backward(self):
        g = self.g
        P = int(g["means"].shape[0])
        dev = g["means"].device
        z = lambda *s: torch.empty(s, dtype=torch.float32, device=dev)  # noqa: E731
        grads = dict(d_means=z(P, 3), d_log_scales=z(P, 3), d_quats=z(P, 4), d_opacity_logits=z(P),
                     d_sh=z(P, g["sh"].shape[1], 3))
        adc = dict(e1=z(P), e2=z(P), e_old=z(P), vis=z(P), gsum=z(P, 2),
                   max_radius=torch.zeros(P, dtype=torch.float32, device=dev))  # max= accumulator
        return grads, adc

    def backward(self, dL_drgb, out=None, stream=None):
        grads, adc = out if out is not None else self.alloc_backward()
        Tf, nc = self._fwd
        render_bwd(self.ctx, dL_drgb, Tf, nc, stream)
        adc_stats(self.ctx, grads, adc, stream)
        return grads, adc
