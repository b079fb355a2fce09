"""NEXT-4: the mini-batch gradient-variance laboratory on the fast path.

Host orchestration only — every numeric step runs in libmvgs.so: for each sampled mini-batch
(a list of view indices, drawn by the caller: the random draw is an input) the batch is
preprocessed, rendered, differentiated against its target photos (mvgs_loss_grad), pushed
back to the Gaussians (mvgs_render_bwd + mvgs_adc_stats) and its ∂L/∂means accumulated
(mvgs_grad_moments); mvgs_grad_variance then evaluates
    𝕍 ≈ (1/K)Σ‖∇φ̄_k‖² − ‖(1/K)Σ∇φ̄_k‖²
with parameters frozen throughout.
"""
from __future__ import annotations

import numpy as np
import torch

from . import mvgs


class VarianceLab:
    def __init__(self, g: dict, cams: np.ndarray, targets: torch.Tensor, loss: int = mvgs.LOSS_L2, device: int = 0):
        self.g = g
        self.cams = np.ascontiguousarray(cams)
        self.targets = targets  # [M,3,H,W] device fp32
        self.loss = loss
        self.R = mvgs.Rasterizer(device)
        P = int(g["means"].shape[0])
        dev = g["means"].device
        self.n = 3 * P
        self.sum = torch.zeros(self.n, dtype=torch.float64, device=dev)
        self.sumsq = torch.zeros(1, dtype=torch.float64, device=dev)
        self.out = torch.zeros(1, dtype=torch.float64, device=dev)
        self.lossv = torch.zeros(1, dtype=torch.float64, device=dev)
        self.K = 0
        self._bufs = {}
        self.auto_reserve = True  # grow capacities on overflow (one host sync per batch); off once sized

    def reset(self):
        self.sum.zero_()
        self.sumsq.zero_()
        self.K = 0

    def _buffers(self, B):
        if B not in self._bufs:
            H, W = int(self.cams[0]["height"]), int(self.cams[0]["width"])
            dev = self.g["means"].device
            f = dict(dtype=torch.float32, device=dev)
            self._bufs[B] = dict(rgb=torch.empty((B, 3, H, W), **f), T=torch.empty((B, H, W), **f),
                                 nc=torch.empty((B, H, W), dtype=torch.int32, device=dev),
                                 dL=torch.empty((B, 3, H, W), **f), tgt=torch.empty((B, 3, H, W), **f))
        return self._bufs[B]

    def batch_gradient(self, views):
        """∂L/∂means of one mini-batch (views: sequence of view indices); returns the grads dict."""
        views = list(views)
        b = self._buffers(len(views))
        self.R.preprocess(self.g, self.cams[views], auto_reserve=self.auto_reserve)
        mvgs.render_fwd(self.R.ctx, b["rgb"], b["T"], b["nc"])
        torch.index_select(self.targets, 0, torch.tensor(views, device=self.targets.device), out=b["tgt"])
        mvgs.loss_grad(self.R.ctx, b["rgb"], b["tgt"], b["dL"], self.loss, loss=self.lossv)
        mvgs.render_bwd(self.R.ctx, b["dL"], b["T"], b["nc"])
        if "grads" not in b:
            b["grads"], b["adc"] = self.R.alloc_backward()
        mvgs.adc_stats(self.R.ctx, b["grads"], b["adc"])
        return b["grads"]

    def add_batch(self, views):
        gr = self.batch_gradient(views)
        mvgs.grad_moments(self.R.ctx, gr["d_means"], self.sum, self.sumsq)
        self.K += 1

    def variance(self) -> float:
        mvgs.grad_variance(self.R.ctx, self.sum, self.sumsq, self.K, self.out)
        return float(self.out.item())

    def run(self, batches) -> float:
        self.reset()
        for b in batches:
            self.add_batch(b)
        return self.variance()
