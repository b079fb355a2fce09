"""Pins for the NEXT-4 oracle (oracle/variance.py): the §4.2 variance estimator.
Closed forms (SPEC S:454 two-sample case), the definition computed two ways, the textbook
finite-population variance of a sample mean against brute-force enumeration of every batch,
and the rasterizer's view independence (a multi-view batch gradient is the mean of the
single-view gradients)."""
import numpy as np

import oracle
import synth
from oracle import variance as ov


def test_two_sample_closed_form():
    msq, sqm, v = ov.estimator([[1.0, 0.0], [0.0, 1.0]])
    # g1 = (1,0), g2 = (0,1): mean ‖g‖² = 1, mean g = (½,½) → ‖·‖² = ½, 𝕍 = ½
    assert msq == 1.0 and sqm == 0.5 and v == 0.5


def test_estimator_identity_against_definition():
    rng = np.random.default_rng(0)
    gs = rng.normal(size=(37, 101)) + rng.normal(size=101)
    _, _, v = ov.estimator(gs)
    np.testing.assert_allclose(v, ov.two_pass_variance(gs), rtol=1e-10)
    assert ov.estimator(np.tile(gs[:1], (5, 1)))[2] < 1e-12  # identical batches → 0


def test_enumeration_equals_finite_population_closed_form():
    rng = np.random.default_rng(1)
    per_view = rng.normal(size=(7, 13)) * rng.uniform(0.5, 2, size=(7, 1))
    for m in range(1, 8):
        np.testing.assert_allclose(ov.exact_subset_variance(per_view, m), ov.finite_population_variance(per_view, m),
                                   rtol=1e-10, atol=1e-14)
    v = [ov.exact_subset_variance(per_view, m) for m in range(1, 8)]
    assert all(a > b for a, b in zip(v, v[1:])) and v[-1] < 1e-12  # strictly decreasing, 0 at m = M


def small_scene(M=4, P=400, W=40, H=32, seed=3):
    cfg = synth.scaled(synth.CONFIGS["tiny"], P=P, V=M, W=W, H=H)
    g, cams = synth.make_scene(cfg, seed=seed)
    targets = synth.make_lab_targets(M, H, W, seed)
    return g, cams, targets


def test_batch_gradient_is_mean_of_view_gradients():
    g, cams, targets = small_scene()
    per_view = ov.view_gradients(g, cams, targets)
    o = oracle.Oracle(g, cams[[0, 2, 3]])
    d = o.forward()["rgb"] - targets[[0, 2, 3]]
    gb = o.backward((2.0 * d / d.size).astype(np.float32))["d_means"].reshape(-1)
    np.testing.assert_allclose(gb, per_view[[0, 2, 3]].mean(0), rtol=1e-5, atol=1e-7 * np.abs(gb).max())


def test_lab_identical_views_zero_variance():
    g, cams, targets = small_scene(M=3)
    cams = cams[[0, 0, 0]]
    targets = targets[[0, 0, 0]]
    _, _, v = ov.lab(g, cams, targets, [[0], [1], [2]])
    assert abs(v) < 1e-15
