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
    """One flat fp32 buffer holding every per-Gaussian output that is summed over views.

    With chunks > 1 the buffer is laid out chunk-major: Gaussians [lo_c, hi_c) (lo_c a
    multiple of 256, the pair-slot block) own one contiguous slice [fields of chunk c], so
    each finished chunk of the per-Gaussian kernel can be all-reduced while the next one
    computes (SURVEY.md §8(e) lever 1).  chunks = 1 is the plain field-major layout."""

    FIELDS = ("d_means", "d_log_scales", "d_quats", "d_opacity_logits", "d_sh", "e1", "e2", "vis")

    def __init__(self, P: int, sh_stride: int, device, chunks: int = 1):
        cg = -(-max(P, 1) // max(chunks, 1))
        cg = -(-cg // 256) * 256
        self.P = P
        self.bounds = [(lo, min(P, lo + cg)) for lo in range(0, max(P, 1), cg)] if P > 0 else [(0, 0)]
        tail = dict(d_means=(3,), d_log_scales=(3,), d_quats=(4,), d_opacity_logits=(), d_sh=(sh_stride, 3),
                    e1=(), e2=(), vis=())
        per_row = sum(int(torch.Size(t).numel()) for t in tail.values())
        self.flat = torch.zeros(per_row * P, dtype=torch.float32, device=device)
        self.chunk_flat, self.chunk_views = [], []
        off = 0
        for lo, hi in self.bounds:
            n = hi - lo
            self.chunk_flat.append(self.flat[off:off + per_row * n])
            views = {}
            for k in self.FIELDS:
                m = n * int(torch.Size(tail[k]).numel())
                views[k] = self.flat[off:off + m].view((n,) + tail[k])
                off += m
            self.chunk_views.append(views)
        self.e_old = torch.zeros(P, dtype=torch.float32, device=device)

    @property
    def views(self) -> dict:
        """Per-field tensors over all Gaussians (views for one chunk, gathered copies otherwise)."""
        if len(self.chunk_views) == 1:
            return self.chunk_views[0]
        return {k: torch.cat([cv[k] for cv in self.chunk_views]) for k in self.FIELDS}

    @property
    def grads(self) -> dict:
        return {k: self.views[k] for k in GRAD_KEYS}

    @property
    def adc(self) -> dict:
        v = self.views
        return dict(e1=v["e1"], e2=v["e2"], vis=v["vis"], e_old=self.e_old)

    def chunk_outputs(self, c: int):
        """(lo, hi, grads, adc) of chunk c: tensors whose row 0 is Gaussian lo."""
        lo, hi = self.bounds[c]
        v = self.chunk_views[c]
        return lo, hi, {k: v[k] for k in GRAD_KEYS}, dict(e1=v["e1"], e2=v["e2"], vis=v["vis"],
                                                           e_old=self.e_old[lo:hi])

    def allreduce(self, group=None):
        import torch.distributed as dist
        dist.all_reduce(self.flat, op=dist.ReduceOp.SUM, group=group)


def adc_stats_allreduce(ctx, buf: GradBuffer, group=None, stream=None, compute=None):
    """S8–S9 chunk by chunk, each chunk's slice all-reduced (async, on NCCL's own stream) as
    soon as its kernel is enqueued, so the collective of chunk c overlaps the kernel of chunk
    c+1; returns once the current stream waits for every reduction.  `compute(c, lo, hi,
    grads, adc)` replaces the library call (host tests of the collective schedule)."""
    import torch.distributed as dist

    if compute is None:
        from . import mvgs

        def compute(c, lo, hi, gr, ad):
            mvgs.adc_stats_range(ctx, lo, hi, gr, ad, stream=stream)
    import contextlib

    # ProcessGroupNCCL orders each collective after torch's CURRENT stream: make the stream the
    # kernels are enqueued on the current one, so a chunk is never reduced before it is written
    if stream is not None and not isinstance(stream, torch.cuda.Stream):
        stream = torch.cuda.ExternalStream(int(stream))  # a raw cudaStream_t handle
    on_stream = torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext()
    works = []
    with on_stream:
        for c in range(len(buf.bounds)):
            lo, hi, gr, ad = buf.chunk_outputs(c)
            if hi > lo:
                compute(c, lo, hi, gr, ad)
            works.append(dist.all_reduce(buf.chunk_flat[c], op=dist.ReduceOp.SUM, group=group, async_op=True))
        for w in works:
            w.wait()
