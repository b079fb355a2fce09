"""ctypes loader for the C oracle (oracle/oracle.c).  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  The product path
(paper_2506_12727_b200) never imports it, and it never imports the product.

See oracle.c's header for what is computed and which PAPER.md passage each
step follows.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "oracle.c")
LIB = os.path.join(HERE, "liboracle.so")
CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-Wall", "-fopenmp"]

NO_EARLY_TERMINATION = 1
NG = 10  # per-pair gradient record: gx gy e1 dA dB dC dO dr dg db


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, SRC, "-o", tmp, "-lm"])
        os.replace(tmp, LIB)
    return LIB


class _Scene(C.Structure):
    _fields_ = [
        ("P", C.c_int64),
        ("sh_degree", C.c_int32),
        ("sh_stride", C.c_int32),
        ("means", C.c_void_p),
        ("log_scales", C.c_void_p),
        ("quats", C.c_void_p),
        ("opacity_logits", C.c_void_p),
        ("sh", C.c_void_p),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build() if LIB == os.path.join(HERE, "liboracle.so") else LIB)
        vp, i64 = C.c_void_p, C.c_int64
        L.oracle_create.restype = vp
        L.oracle_create.argtypes = [C.POINTER(_Scene), vp, C.c_int, vp, C.c_int]
        L.oracle_create_masked.restype = vp
        L.oracle_create_masked.argtypes = [C.POINTER(_Scene), vp, C.c_int, vp, C.c_int, vp]
        L.oracle_destroy.argtypes = [vp]
        L.oracle_forward.argtypes = [vp]
        L.oracle_backward.argtypes = [vp, vp]
        L.oracle_num_entries.restype = i64
        L.oracle_num_entries.argtypes = [vp]
        L.oracle_phase_times.argtypes = [vp, vp]
        L.oracle_get_depth.argtypes = [vp, vp]
        L.oracle_get_nblend.argtypes = [vp, vp]
        L.oracle_decision_hash.restype = C.c_uint64
        L.oracle_decision_hash.argtypes = [vp]
        for name, n in [("oracle_get_image", 3), ("oracle_get_image32", 3), ("oracle_get_lists", 2), ("oracle_get_pairs", 3),
                        ("oracle_get_opacity32", 1), ("oracle_get_pair_grads", 1), ("oracle_get_grads", 9)]:
            getattr(L, name).argtypes = [vp] + [vp] * n
        L.oracle_set_threads.argtypes = [C.c_int]
        L.oracle_get_threads.restype = C.c_int
        L.oracle_ca_exp.restype = C.c_float
        L.oracle_ca_exp.argtypes = [C.c_float]
        L.oracle_adc_example.argtypes = [C.c_int, vp, vp, vp, vp]
        _lib = L
    return _lib


def set_threads(n: int) -> None:
    """Host threads of the oracle (1, the default, runs every loop in its written order; more
    is only for the CPU timing baseline — bench.py's cpu_baseline / --impl reference)."""
    lib().oracle_set_threads(int(n))


def get_threads() -> int:
    return int(lib().oracle_get_threads())


def use_library(path: str | None = None):
    """Load the oracle from another build of oracle.c (mutation tests), or back from the
    default build with path=None."""
    global _lib
    _lib = None
    if path is not None:
        global LIB
        saved = LIB
        LIB = path
        try:
            lib()
        finally:
            LIB = saved
    return lib()


def build_variant(src_text: str, out: str) -> str:
    """Compile a modified copy of oracle.c (mutation tests) with the oracle's flags."""
    import tempfile
    with tempfile.NamedTemporaryFile("w", suffix=".c", delete=False) as f:
        f.write(src_text)
    subprocess.check_call(["gcc", *CFLAGS, f.name, "-o", out, "-lm"])
    os.unlink(f.name)
    return out


def _p(a):
    return None if a is None else a.ctypes.data


def ca_exp(x: float) -> np.float32:
    return np.float32(lib().oracle_ca_exp(float(np.float32(x))))


def adc_example(views, gx, gy):
    """(E_old, E1, E2) of one Gaussian from labelled per-pixel NDC gradients."""
    v = np.ascontiguousarray(views, np.int32)
    x = np.ascontiguousarray(gx, np.float64)
    y = np.ascontiguousarray(gy, np.float64)
    out = np.zeros(3)
    lib().oracle_adc_example(len(v), _p(v), _p(x), _p(y), _p(out))
    return out


class Oracle:
    """One oracle run over a scene and a batch of views.

    ``Oracle(g, cams, bg)`` runs O1–O4 (projection, lists, sort);
    ``forward()`` runs O5; ``backward(dLdC)`` runs O5–O8.
    """

    def __init__(self, g: dict, cams: np.ndarray, bg=(0.0, 0.0, 0.0), flags: int = 0, tile_mask=None):
        self._keep = {k: np.ascontiguousarray(g[k], np.float32)
                      for k in ("means", "log_scales", "quats", "opacity_logits", "sh")}
        self.P = int(self._keep["means"].shape[0])
        self.sh_stride = int(self._keep["sh"].shape[1]) if self.P else 1
        self.sh_degree = int(g["sh_degree"])
        self.cams = np.ascontiguousarray(cams)
        self.V = len(self.cams)
        self.W = int(self.cams[0]["width"])
        self.H = int(self.cams[0]["height"])
        self.TX, self.TY = (self.W + 15) // 16, (self.H + 15) // 16
        self.T = self.TX * self.TY
        self.bg = np.ascontiguousarray(bg, np.float32)
        sc = _Scene(self.P, self.sh_degree, self.sh_stride,
                    *[self._keep[k].ctypes.data for k in ("means", "log_scales", "quats", "opacity_logits", "sh")])
        self.tile_mask = None if tile_mask is None else np.ascontiguousarray(tile_mask, np.uint8).reshape(-1)
        if self.tile_mask is not None:
            assert self.tile_mask.size == self.V * self.T
        self._h = lib().oracle_create_masked(C.byref(sc), self.cams.ctypes.data, self.V, _p(self.bg), flags,
                                             _p(self.tile_mask))
        if not self._h:
            raise ValueError("oracle_create rejected the input")
        self.K = int(lib().oracle_num_entries(self._h))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().oracle_destroy(h)
            self._h = None

    def forward(self):
        lib().oracle_forward(self._h)
        self._rendered = True
        return self.image()

    def phase_times(self):
        """Seconds: (projection O1–O2, lists O3–O4, per-pixel O5–O6, per-Gaussian O7–O8)."""
        out = np.zeros(4)
        lib().oracle_phase_times(self._h, _p(out))
        return out

    def decision_hash(self) -> int:
        return int(lib().oracle_decision_hash(self._h))

    def backward(self, dLdC: np.ndarray):
        d = np.ascontiguousarray(dLdC, np.float32)
        assert d.shape == (self.V, 3, self.H, self.W)
        lib().oracle_backward(self._h, _p(d))
        self._rendered = True
        return self.grads()

    def image(self):
        if not getattr(self, "_rendered", False):
            raise RuntimeError("Oracle.image() before forward()/backward()")
        rgb = np.zeros((self.V, 3, self.H, self.W))
        Tf = np.zeros((self.V, self.H, self.W))
        nc = np.zeros((self.V, self.H, self.W), np.int32)
        lib().oracle_get_image(self._h, _p(rgb), _p(Tf), _p(nc))
        return dict(rgb=rgb, T_final=Tf, n_contrib=nc)

    def image32(self):
        """The last forward's image / T_final in fp32 canonical arithmetic: the
        decision chain's T and α, C = fma(rgb32, α·T, C) in list order, out = fma(T, bg, C)."""
        rgb = np.zeros((self.V, 3, self.H, self.W), np.float32)
        Tf = np.zeros((self.V, self.H, self.W), np.float32)
        x = np.zeros((self.V, 3, self.H, self.W))
        lib().oracle_get_image32(self._h, _p(rgb), _p(Tf), _p(x))
        return dict(rgb=rgb, T_final=Tf, rgb_x=x)

    def nblend(self):
        """Blended entries per pixel [V,H,W] of the last forward."""
        n = np.zeros((self.V, self.H, self.W), np.int32)
        lib().oracle_get_nblend(self._h, _p(n))
        return n

    def depth(self):
        """Predicted depth Σ dᵢαᵢTᵢ [V,H,W] of the last forward (fp64)."""
        d = np.zeros((self.V, self.H, self.W))
        lib().oracle_get_depth(self._h, _p(d))
        return d

    def lists(self):
        off = np.zeros(self.V * self.T + 1, np.int64)
        gid = np.zeros(max(self.K, 1), np.int32)
        lib().oracle_get_lists(self._h, _p(off), _p(gid))
        return off, gid[: self.K]

    def pairs(self):
        n = self.V * self.P
        ints = np.zeros((self.V, self.P, 9), np.int32)
        flts = np.zeros((self.V, self.P, 6), np.float32)
        rgb = np.zeros((self.V, self.P, 3))
        if n:
            lib().oracle_get_pairs(self._h, _p(ints), _p(flts), _p(rgb))
        names = ["zvis", "vis", "radius", "rx0", "ry0", "rx1", "ry1", "tiles", "clamp"]
        out = {k: ints[..., j] for j, k in enumerate(names)}
        out.update({k: flts[..., j] for j, k in enumerate(["depth", "px", "py", "A", "B", "C"])})
        out["rgb"] = rgb
        o = np.zeros(self.P, np.float32)
        lib().oracle_get_opacity32(self._h, _p(o))
        out["opacity"] = o
        return out

    def pair_grads(self):
        out = np.zeros((self.V, self.P, NG))
        lib().oracle_get_pair_grads(self._h, _p(out))
        return out

    def grads(self):
        P, S = self.P, self.sh_stride
        o = dict(d_means=np.zeros((P, 3)), d_log_scales=np.zeros((P, 3)), d_quats=np.zeros((P, 4)),
                 d_opacity_logits=np.zeros(P), d_sh=np.zeros((P, S, 3)), e1=np.zeros(P), e2=np.zeros(P),
                 e_old=np.zeros(P), vis=np.zeros(P))
        lib().oracle_get_grads(self._h, *[_p(o[k]) for k in ("d_means", "d_log_scales", "d_quats",
                                                             "d_opacity_logits", "d_sh", "e1", "e2", "e_old", "vis")])
        return o

    def adc_extra(self):
        """max_radius [P]: SPEC S:248's max_screen_radius, the largest radius (R7) over the views
        where the pair covers a tile; gsum [P,2]: Σ over views and pixels of ∇_{p_i}L, the vector
        whose norm is E_old.  From the last backward; small scenes only (per-pair arrays)."""
        pr = self.pairs()
        rad = np.where(pr["tiles"] > 0, pr["radius"], 0)
        mr = rad.max(axis=0).astype(np.float64) if self.V else np.zeros(self.P)
        return dict(max_radius=mr, gsum=self.pair_grads()[:, :, 0:2].sum(axis=0))


def run(g, cams, bg=(0.0, 0.0, 0.0), dLdC=None, flags=0):
    """Convenience: full oracle pass; returns (Oracle, image dict, grads dict|None)."""
    o = Oracle(g, cams, bg, flags)
    if dLdC is None:
        return o, o.forward(), None
    gr = o.backward(dLdC)
    return o, o.image(), gr
