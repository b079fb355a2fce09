"""Measured D-SSIM gradient error vs the oracle (the floor a 1e-3 / 1e-4 relative rule needs): the
evidence behind tests/test_gpu_dssim.py's tolerance.  Run on a GPU box."""
import sys, numpy as np
import os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import synth
from oracle import dssim
from test_gpu_dssim import gpu_dssim
for shape in [(2, 45, 61), (1, 16, 16), (1, 7, 5), (1, 96, 128)]:
    V, H, W = shape
    img, tgt, depth, Tf, cams = synth.make_dssim_inputs(V, H, W, seed=H + W)
    loss, g = gpu_dssim(img, tgt, depth, Tf, cams)
    ref_loss, ref = dssim.dssim3d(img, tgt, depth, Tf, cams)
    d = np.abs(g - ref); mx = np.abs(ref).max()
    # smallest (a, b) with |Δ| ≤ a|ref| + b·max|ref|: report the needed floor for a = 1e-3 and 1e-4
    for a in (1e-3, 1e-4):
        need = np.max(np.maximum(d - a * np.abs(ref), 0)) / mx
        print(shape, f"rel {a}: floor needed {need:.2e}", end="; ")
    print("loss |Δ|", abs(loss - ref_loss), "tensor rel", np.linalg.norm(g - ref) / np.linalg.norm(ref))
