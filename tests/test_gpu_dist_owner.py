"""Multi-GPU exchanges emulated on one GPU: N ranks = N contexts, each
rendering its view_shard of the batch; the exchange is replayed with device copies in the
order the real plan issues it.  Against one context rendering all views:
  * owner-sharded (lever 3): every owner's S8–S9 over all views equals the single-GPU rows of
    its range — gradients, E1, E2 and E_old (exact definitions, no per-rank approximation),
    vis and max_radius bit-exact;
  * all-reduce: the summed per-rank buffers plus E_old = ‖Σ gsum‖ equal the single GPU."""
import numpy as np
import pytest
import torch

import synth
from gpu_harness import to_dev

pytestmark = pytest.mark.gpu


def _scene():
    cfg = synth.scaled(synth.CONFIGS["tiny"], P=6000, V=6)
    g, cams = synth.make_scene(cfg)
    dL = synth.make_dLdC_scaled(cfg.V, cfg.H, cfg.W, 5)
    return g, cams, dL


def _render(g, cams, dL):
    from paper_2506_12727_b200 import mvgs
    R = mvgs.Rasterizer(0)
    R.preprocess(to_dev(g), cams)
    R.forward()
    mvgs.render_bwd(R.ctx, torch.from_numpy(dL).cuda(), *R._fwd)
    return R


def _outputs(P, S, dev="cuda"):
    z = lambda *s: torch.zeros(s, dtype=torch.float32, device=dev)  # noqa: E731
    grads = dict(d_means=z(P, 3), d_log_scales=z(P, 3), d_quats=z(P, 4), d_opacity_logits=z(P), d_sh=z(P, S, 3))
    adc = dict(e1=z(P), e2=z(P), e_old=z(P), vis=z(P), gsum=z(P, 2), max_radius=z(P))
    return grads, adc


def _close(got, ref, name):
    got, ref = got.cpu().numpy().astype(np.float64), ref.cpu().numpy().astype(np.float64)
    scale = max(np.abs(ref).max(), 1e-30)
    rel = np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30)
    assert rel <= 1e-5, f"{name}: rel {rel}"
    assert np.all(np.abs(got - ref) <= 1e-4 * np.abs(ref) + 1e-6 * scale), name


@pytest.mark.parametrize("world", [2, 3])
def test_owner_sharded_equals_single_gpu(require_gpu, world):
    from paper_2506_12727_b200 import mvgs
    from paper_2506_12727_b200.dist import exchange_plan, owner_bounds, view_renderer, view_shard
    g, cams, dL = _scene()
    V, P, S = len(cams), g["means"].shape[0], g["sh"].shape[1]
    full = _render(g, cams, dL)
    ref_g, ref_a = _outputs(P, S)
    mvgs.adc_stats(full.ctx, ref_g, ref_a)
    bounds = owner_bounds(P, world)
    renderer = view_renderer(V, world)
    ranks, offs = [], []
    for r in range(world):
        lo, hi = view_shard(V, world, r)
        R = _render(g, cams[lo:hi], dL[lo:hi])
        slot_off, slots = mvgs.owner_slices(R.ctx, bounds, hi - lo)
        view_off, recv = mvgs.owner_prepare(R.ctx, cams, int(bounds[r]), int(bounds[r + 1]))
        ranks.append((R, slots, recv, lo))
        offs.append((slot_off, view_off))
    # replay every rank's plan: local copies, and each send delivered into its owner's receive slice
    for r in range(world):
        R, slots, recv, lo = ranks[r]
        sends, local, _ = exchange_plan(r, world, renderer, *offs[r])
        for a, b, ra, rb in local:
            assert b - a == rb - ra
            recv[ra * 12:rb * 12].copy_(slots[a * 12:b * 12])
        mine = [v for v in range(V) if renderer[v] == r]
        for l, v in enumerate(mine):
            for o in range(world):
                if o == r:
                    continue
                a, b = offs[r][0][l, o], offs[r][0][l, o + 1]
                ra, rb = offs[o][1][v], offs[o][1][v + 1]
                assert b - a == rb - ra, (r, o, v)
                ranks[o][2][ra * 12:rb * 12].copy_(slots[a * 12:b * 12])
    torch.cuda.synchronize()
    for o in range(world):
        lo_g, hi_g = int(bounds[o]), int(bounds[o + 1])
        gr, ad = _outputs(hi_g - lo_g, S)
        mvgs.owner_adc_stats(ranks[o][0].ctx, gr, ad)
        torch.cuda.synchronize()
        for k in gr:
            _close(gr[k], ref_g[k][lo_g:hi_g], f"{k} owner {o}")
        for k in ("e1", "e2", "e_old", "gsum"):
            _close(ad[k], ref_a[k][lo_g:hi_g], f"{k} owner {o}")
        assert torch.equal(ad["vis"], ref_a["vis"][lo_g:hi_g])
        assert torch.equal(ad["max_radius"], ref_a["max_radius"][lo_g:hi_g])


def test_allreduce_emulation_equals_single_gpu(require_gpu):
    from paper_2506_12727_b200 import mvgs
    from paper_2506_12727_b200.dist import GradBuffer, view_shard
    g, cams, dL = _scene()
    V, P, S = len(cams), g["means"].shape[0], g["sh"].shape[1]
    full = _render(g, cams, dL)
    ref_g, ref_a = _outputs(P, S)
    mvgs.adc_stats(full.ctx, ref_g, ref_a)
    total = GradBuffer(P, S, "cuda", chunks=3)
    for r in range(2):
        lo, hi = view_shard(V, 2, r)
        R = _render(g, cams[lo:hi], dL[lo:hi])
        b = GradBuffer(P, S, "cuda", chunks=3)
        for c in range(len(b.bounds)):
            a0, a1, gr, ad = b.chunk_outputs(c)
            mvgs.adc_stats_range(R.ctx, a0, a1, gr, {k: v for k, v in ad.items() if k != "e_old"})
        total.flat += b.flat  # what the all-reduce sums
    for c in range(len(total.bounds)):
        a0, a1, _, ad = total.chunk_outputs(c)
        mvgs.e_old_from_gsum(full.ctx, ad["gsum"], ad["e_old"])
    torch.cuda.synchronize()
    for k in ref_g:
        _close(total.grads[k], ref_g[k], k)
    adc = total.adc
    for k in ("e1", "e2", "e_old", "gsum"):
        _close(adc[k], ref_a[k], k)
    assert torch.equal(adc["vis"], ref_a["vis"])
