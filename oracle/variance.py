"""Oracle for NEXT-4: the mini-batch gradient-variance laboratory.
TEST INFRASTRUCTURE ONLY (same import rules as oracle/__init__.py).

Definitions followed, in fp64:
  𝕍(x) := E‖x − μ‖²,  μ = E x                                                  (Eq. vector_variance)
  𝕍 ≈ (1/|S̃|)Σ‖∇φ̄_k‖² − ‖(1/|S̃|)Σ∇φ̄_k‖²  over sampled mini-batches B_k
  ∇φ̄_k = (1/|B_k|)Σ_{i∈B_k}∇φ_i
Readings: a data point i is one view (its per-pixel loss averaged over the
view's pixels), so ∇φ̄_k of a batch of m views is the gradient of the loss averaged over the
batch's pixels; the frozen parameter vector is the Gaussian means; the loss is ℓ2
for parity (continuous in C) or ℓ1 (the training loss).
"""
from __future__ import annotations

import itertools

import numpy as np


def estimator(gs):
    """(mean ‖g‖², ‖mean g‖², 𝕍) of the rows of gs [K, n] — P:152–156 term by term."""
    gs = np.asarray(gs, np.float64)
    msq = float(np.mean(np.sum(gs * gs, axis=1)))
    mu = gs.mean(axis=0)
    sqm = float(mu @ mu)
    return msq, sqm, msq - sqm


def two_pass_variance(gs):
    """E‖g − μ‖² directly from the definition."""
    gs = np.asarray(gs, np.float64)
    d = gs - gs.mean(axis=0)
    return float(np.mean(np.sum(d * d, axis=1)))


def batch_gradient(per_view, subset):
    """∇φ̄_k = mean of the per-view gradients of the batch."""
    return np.asarray(per_view, np.float64)[list(subset)].mean(axis=0)


def exact_subset_variance(per_view, m):
    """𝕍 over ALL C(M, m) batches of m distinct views, each equally likely (brute force)."""
    M = len(per_view)
    gs = [batch_gradient(per_view, s) for s in itertools.combinations(range(M), m)]
    return two_pass_variance(np.stack(gs))


def finite_population_variance(per_view, m):
    """Textbook closed form of the variance of a sample mean drawn without replacement:
    𝕍(m) = (σ²/m)·(M − m)/(M − 1),  σ² = (1/M)Σ‖g_i − ḡ‖²  (Lemma 1's 1/m law, P:329–424,
    with the finite-population correction)."""
    g = np.asarray(per_view, np.float64)
    M = len(g)
    s2 = two_pass_variance(g)
    return s2 / m * (M - m) / (M - 1) if M > 1 else 0.0


def view_gradients(g, cams, targets, loss="l2"):
    """Per-view ∇φ_i over the means with the oracle rasterizer: loss of view i = mean over its
    3·H·W values of (C − C*)² (ℓ2) or |C − C*| (ℓ1)."""
    import oracle
    out = []
    for i in range(len(cams)):
        o = oracle.Oracle(g, cams[i:i + 1])
        im = o.forward()["rgb"]
        d = im - targets[i:i + 1]
        n = d.size
        dL = (2.0 * d / n) if loss == "l2" else (np.sign(d) / n)
        out.append(o.backward(dL.astype(np.float32))["d_means"].reshape(-1).astype(np.float64))
    return np.stack(out)


def lab(g, cams, targets, batches, loss="l2"):
    """The §4.2 Monte-Carlo estimate over the given batches (lists of view indices), each
    batch rendered and differentiated as one multi-view batch by the oracle rasterizer."""
    import oracle
    gs = []
    for b in batches:
        o = oracle.Oracle(g, cams[list(b)])
        im = o.forward()["rgb"]
        d = im - targets[list(b)]
        n = d.size
        dL = (2.0 * d / n) if loss == "l2" else (np.sign(d) / n)
        gs.append(o.backward(dL.astype(np.float32))["d_means"].reshape(-1).astype(np.float64))
    return estimator(np.stack(gs))
