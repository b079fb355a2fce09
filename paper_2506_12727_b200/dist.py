"""View-sharded data parallelism.

Every output of the path is a sum over the batch's views — the multi-view mini-batch
gradient, E1 and E2, the `vis` denominator and gsum =
Σ_views Σ∇ (R49), whose norm is E_old — so ranks render disjoint blocks of
views against full replicas of the Gaussians and one exchange completes the step.  Two
exchanges are provided:

* all-reduce (SURVEY §8(e) levers 1): ONE flat fp32 buffer [d_means | d_log_scales | d_quats |
  d_opacity_logits | d_sh | e1 | e2 | vis | gsum], chunk-major so each chunk of the
  per-Gaussian kernel is all-reduced (NCCL over NVLink/NVSwitch) while the next computes;
  E_old = ‖gsum‖ after the sum, so it is the single-GPU E_old;
* owner-sharded (lever 3): each per-pair gradient slot (48 B) goes to the rank that owns its
  Gaussian (contiguous ranges of 256-Gaussian blocks); the owner runs S8–S9 over all views and
  holds the full sums for its range (reduce-scatter semantics).  Per rank it moves
  (N−1)/N · 48 B per pair of its views instead of 2(N−1)/N · 4·(11+S+5) B per Gaussian.

Host-side plumbing only: buffer layout, view partition, exchange plans and the collective
calls; every value is computed by libmvgs kernels.
"""
from __future__ import annotations

import contextlib

import numpy as np
import torch

GRAD_KEYS = ("d_means", "d_log_scales", "d_quats", "d_opacity_logits", "d_sh")
ADC_KEYS = ("e1", "e2", "vis", "gsum")
PG_STRIDE = 12  # floats per per-pair gradient slot


def view_shard(n_views: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block [lo, hi) of views for `rank` (sizes differ by at most one)."""
    base, extra = divmod(n_views, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def view_renderer(n_views: int, world: int) -> list[int]:
    """The rank that renders each view under view_shard."""
    out = []
    for r in range(world):
        lo, hi = view_shard(n_views, world, r)
        out += [r] * (hi - lo)
    return out


def owner_bounds(P: int, world: int) -> np.ndarray:
    """[world+1] Gaussian bounds of the owner ranges: contiguous, multiples of 256 (the pair-slot
    block), as equal as the blocks allow; bounds[-1] = P."""
    nb = -(-max(P, 0) // 256)
    per = -(-nb // world) if world else 0
    b = [min(P, r * per * 256) for r in range(world)] + [P]
    return np.asarray(b, np.int64)


class GradBuffer:
    """One flat fp32 buffer holding every per-Gaussian output that is summed over views.

    With chunks > 1 the buffer is laid out chunk-major: Gaussians [lo_c, hi_c) (lo_c a
    multiple of 256, the pair-slot block) own one contiguous slice [fields of chunk c], so
    each finished chunk of the per-Gaussian kernel can be all-reduced while the next one
    computes (SURVEY.md §8(e) lever 1).  chunks = 1 is the plain field-major layout."""

    # gsum first: every chunk starts at an even offset (chunks are multiples of 256 rows), so the
    # float2 loads of the E_old kernel are 8-byte aligned
    FIELDS = ("gsum", "d_means", "d_log_scales", "d_quats", "d_opacity_logits", "d_sh", "e1", "e2", "vis")

    def __init__(self, P: int, sh_stride: int, device, chunks: int = 1):
        cg = -(-max(P, 1) // max(chunks, 1))
        cg = -(-cg // 256) * 256
        self.P = P
        self.bounds = [(lo, min(P, lo + cg)) for lo in range(0, max(P, 1), cg)] if P > 0 else [(0, 0)]
        tail = dict(d_means=(3,), d_log_scales=(3,), d_quats=(4,), d_opacity_logits=(), d_sh=(sh_stride, 3),
                    e1=(), e2=(), vis=(), gsum=(2,))
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
        return dict(e1=v["e1"], e2=v["e2"], vis=v["vis"], gsum=v["gsum"], e_old=self.e_old)

    def chunk_outputs(self, c: int):
        """(lo, hi, grads, adc) of chunk c: tensors whose row 0 is Gaussian lo."""
        lo, hi = self.bounds[c]
        v = self.chunk_views[c]
        return lo, hi, {k: v[k] for k in GRAD_KEYS}, dict(e1=v["e1"], e2=v["e2"], vis=v["vis"], gsum=v["gsum"],
                                                           e_old=self.e_old[lo:hi])

    def allreduce(self, group=None):
        import torch.distributed as dist
        dist.all_reduce(self.flat, op=dist.ReduceOp.SUM, group=group)


def _on_stream(stream):
    # ProcessGroupNCCL orders each collective after torch's CURRENT stream: make the stream the
    # kernels are enqueued on the current one, so data is never exchanged before it is written
    if stream is not None and not isinstance(stream, torch.cuda.Stream):
        stream = torch.cuda.ExternalStream(int(stream))  # a raw cudaStream_t handle
    return torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext()


def adc_stats_allreduce(ctx, buf: GradBuffer, group=None, stream=None, compute=None, e_old=None):
    """S8–S9 chunk by chunk, each chunk's slice all-reduced (async, on NCCL's own stream) as
    soon as its kernel is enqueued, so the collective of chunk c overlaps the kernel of chunk
    c+1; then E_old = ‖Σ gsum‖ per chunk (the single-GPU E_old).  Returns once the current
    stream waits for every reduction.  `compute(c, lo, hi, grads, adc)` replaces the library
    call and `e_old(c, lo, hi, gsum, e_old)` the E_old kernel (host tests of the schedule)."""
    import torch.distributed as dist

    if compute is None or e_old is None:
        from . import mvgs
    if compute is None:
        def compute(c, lo, hi, gr, ad):
            mvgs.adc_stats_range(ctx, lo, hi, gr, ad, stream=stream)
    if e_old is None:
        def e_old(c, lo, hi, gs, eo):
            mvgs.e_old_from_gsum(ctx, gs, eo, stream=stream)
    works = []
    with _on_stream(stream):
        for c in range(len(buf.bounds)):
            lo, hi, gr, ad = buf.chunk_outputs(c)
            if hi > lo:
                compute(c, lo, hi, gr, {k: v for k, v in ad.items() if k != "e_old"})
            works.append(dist.all_reduce(buf.chunk_flat[c], op=dist.ReduceOp.SUM, group=group, async_op=True))
        for c, w in enumerate(works):
            w.wait()
            lo, hi, _, ad = buf.chunk_outputs(c)
            if hi > lo:
                e_old(c, lo, hi, ad["gsum"], ad["e_old"])


# ----------------------------------------------------------------------- owner-sharded (lever 3)
def exchange_plan(rank: int, world: int, renderer: list[int], slot_off: np.ndarray, view_off: np.ndarray):
    """The point-to-point plan of one rank.  slot_off [V_r, world+1]: owner o's slots of this
    rank's local view l are [slot_off[l, o], slot_off[l, o+1]) of its slot array; view_off
    [V_all+1]: global view v's slots of THIS rank's Gaussians go to [view_off[v], view_off[v+1])
    of its receive array.  Returns (sends [(dst, a, b)], local copies [(a, b, ra, rb)],
    receives [(src, ra, rb)]), all in slots, in a fixed order both sides agree on."""
    mine = [v for v, r in enumerate(renderer) if r == rank]
    sends, local, recvs = [], [], []
    for l, v in enumerate(mine):
        for o in range(world):
            a, b = int(slot_off[l, o]), int(slot_off[l, o + 1])
            if o == rank:
                local.append((a, b, int(view_off[v]), int(view_off[v + 1])))
            elif b > a:
                sends.append((o, a, b))
    for v, r in enumerate(renderer):
        ra, rb = int(view_off[v]), int(view_off[v + 1])
        if r != rank and rb > ra:
            recvs.append((r, ra, rb))
    return sends, local, recvs


def run_exchange(plan, slots: torch.Tensor, recv: torch.Tensor, group=None):
    """Issue the plan: local slices copied, the rest as one batch of isend/irecv (NCCL over
    NVLink on GPUs, gloo in the host tests).  Tensors are flat fp32, PG_STRIDE floats per slot."""
    import torch.distributed as dist

    sends, local, recvs = plan
    for a, b, ra, rb in local:
        if b - a != rb - ra:
            raise RuntimeError(f"owner exchange: local slice {b - a} slots, layout expects {rb - ra}")
        recv[ra * PG_STRIDE:rb * PG_STRIDE].copy_(slots[a * PG_STRIDE:b * PG_STRIDE])
    ops = [dist.P2POp(dist.isend, slots[a * PG_STRIDE:b * PG_STRIDE], o, group) for o, a, b in sends]
    ops += [dist.P2POp(dist.irecv, recv[ra * PG_STRIDE:rb * PG_STRIDE], r, group) for r, ra, rb in recvs]
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()


def check_plan_sizes(rank: int, world: int, renderer: list[int], slot_off: np.ndarray, view_off: np.ndarray,
                     device, group=None):
    """Every sender's slice length must equal its owner's layout (the same participation
    decisions on both sides); one small all-gather of the per-(view, owner) counts checks it,
    so a mismatch raises instead of desynchronising the point-to-point exchange."""
    import torch.distributed as dist

    V = len(renderer)
    mine = [v for v, r in enumerate(renderer) if r == rank]
    sent = torch.zeros((V, world), dtype=torch.int64, device=device)
    for l, v in enumerate(mine):
        sent[v] = torch.as_tensor(np.diff(slot_off[l]), dtype=torch.int64)
    expect = torch.zeros((V, world), dtype=torch.int64, device=device)
    expect[:, rank] = torch.as_tensor(np.diff(view_off), dtype=torch.int64)
    both = torch.stack([sent, expect])
    dist.all_reduce(both, op=dist.ReduceOp.SUM, group=group)
    if not torch.equal(both[0], both[1]):
        raise RuntimeError("owner exchange: slice sizes disagree between renderer and owner")


def adc_stats_owner(ctx, P: int, cams_all, rank: int, world: int, grads: dict, adc: dict, group=None,
                    stream=None, check: bool = True):
    """S8–S9 with the owner-sharded exchange: after mvgs_render_bwd of this rank's views
    (view_shard of the batch cams_all), send every slot to its owner, receive this rank's Gaussians'
    slots of all views, and run S8–S9 for the owned range over all views.  `grads` / `adc`
    address the owned rows (row 0 = Gaussian owner_bounds(P, world)[rank]).  Returns the
    owned range (lo, hi)."""
    from . import mvgs

    bounds = owner_bounds(P, world)
    renderer = view_renderer(len(cams_all), world)
    n_local = sum(1 for r in renderer if r == rank)
    with _on_stream(stream):
        slot_off, slots = mvgs.owner_slices(ctx, bounds, n_local, stream=stream)
        view_off, recv = mvgs.owner_prepare(ctx, cams_all, int(bounds[rank]), int(bounds[rank + 1]), stream=stream)
        if check and world > 1:
            check_plan_sizes(rank, world, renderer, slot_off, view_off, slots.device, group)
        run_exchange(exchange_plan(rank, world, renderer, slot_off, view_off), slots, recv, group)
        mvgs.owner_adc_stats(ctx, grads, adc, stream=stream)
    return int(bounds[rank]), int(bounds[rank + 1])
