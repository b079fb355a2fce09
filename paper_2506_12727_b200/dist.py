"""View-sharded data parallelism.

Every output of the path is a sum over the batch's views — the multi-view
mini-batch gradient, E1 and E2 and the
`vis` denominator — so ranks render disjoint blocks of views against full
replicas of the Gaussians and ONE all-reduce (NCCL over NVLink/NVSwitch) of a
flat fp32 buffer [d_means | d_log_scales | d_quats | d_opacity_logits | d_sh |
e1 | e2 | vis] completes the step.  E_old = ‖Σ_views Σ∇‖ is not additive; in
multi-GPU mode it stays per rank.

Host-side plumbing only: buffer layout, view partition and the collective call.
"""
from __future__ import annotations

import torch

GRAD_KEYS = ("d_means", "d_log_scales", "d_quats", "d_opacity_logits", "d_sh")
ADC_KEYS = ("e1", "e2", "vis")


def view_shard(n_views: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block [lo, hi) of views for `rank` (sizes differ by at most one)."""
    base, extra = divmod(n_views, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


class GradBuffer:
    """One flat fp32 buffer holding every per-Gaussian output that is summed over views."""

    def __init__(self, P: int, sh_stride: int, device):
        shapes = dict(d_means=(P, 3), d_log_scales=(P, 3), d_quats=(P, 4), d_opacity_logits=(P,),
                      d_sh=(P, sh_stride, 3), e1=(P,), e2=(P,), vis=(P,))
        sizes = {k: int(torch.Size(s).numel()) for k, s in shapes.items()}
        self.flat = torch.zeros(sum(sizes.values()), dtype=torch.float32, device=device)
        self.views, off = {}, 0
        for k, n in sizes.items():
            self.views[k] = self.flat[off:off + n].view(shapes[k])
            off += n
        self.e_old = torch.zeros(P, dtype=torch.float32, device=device)

    @property
    def grads(self) -> dict:
        return {k: self.views[k] for k in GRAD_KEYS}

    @property
    def adc(self) -> dict:
        return dict(e1=self.views["e1"], e2=self.views["e2"], vis=self.views["vis"], e_old=self.e_old)

    def allreduce(self, group=None):
        import torch.distributed as dist
        dist.all_reduce(self.flat, op=dist.ReduceOp.SUM, group=group)
