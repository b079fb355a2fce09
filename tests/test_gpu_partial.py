"""NEXT-1 parity: partial rendering (Alg. 3).  Every
listed pixel of every (view, tile) must equal the full render at that pixel
(n_contrib bit-exact, colour/T ≤ 1e-5 vs the oracle), the thread-efficient and
masked launch shapes must agree bit for bit, and the backward with ∂L/∂C given
at the listed pixels must equal the oracle's backward with ∂L/∂C zero elsewhere
(DESIGN.md §5 rules)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_harness import assert_close_rel, per_view_scale, to_dev

pytestmark = pytest.mark.gpu


def sample_lists(V, T, S, seed):
    rng = np.random.default_rng(seed)
    return np.stack([np.stack([rng.choice(256, S, replace=False) for _ in range(T)]) for _ in range(V)]).astype(np.int32)


def dense_index(pix, TX, H, W):
    """(v, y, x) of every listed pixel, and whether it is inside the image."""
    V, T, S = pix.shape
    v = np.repeat(np.arange(V), T * S).reshape(V, T, S)
    t = np.repeat(np.arange(T)[None, :, None], V, 0).repeat(S, 2)
    y = (t // TX) * 16 + pix // 16
    x = (t % TX) * 16 + pix % 16
    return v, y, x, (x < W) & (y < H)


def run_partial(g, cams, pix, mode, dL_s=None):
    from paper_2506_12727_b200 import mvgs
    R = mvgs.Rasterizer(0)
    R.preprocess(to_dev(g), cams)
    V, T, S = pix.shape
    dev = torch.device("cuda")
    p = torch.from_numpy(pix).to(dev)
    rgb = torch.empty((V, T, S, 3), device=dev)
    Tf = torch.empty((V, T, S), device=dev)
    nc = torch.empty((V, T, S), dtype=torch.int32, device=dev)
    mvgs.render_fwd_partial(R.ctx, p, S, mode, rgb, Tf, nc)
    out = dict(stats=R.stats, occ=mvgs.query(R.ctx))
    if dL_s is not None:
        grads, adc = R.alloc_backward()
        mvgs.render_bwd_partial(R.ctx, p, S, mode, torch.from_numpy(dL_s).to(dev), Tf, nc)
        mvgs.adc_stats(R.ctx, grads, adc)
        out.update({k: v.cpu().numpy() for k, v in grads.items()})
        out.update({k: v.cpu().numpy() for k, v in adc.items()})
    torch.cuda.synchronize()
    out.update(rgb=rgb.cpu().numpy(), T_final=Tf.cpu().numpy(), n_contrib=nc.cpu().numpy())
    del R
    return out


@pytest.fixture(scope="module")
def scene(require_gpu):
    cfg = synth.scaled(synth.CONFIGS["garden"], P=20_000, V=4, W=203, H=137)
    g, cams = synth.make_scene(cfg)
    V, W, H = 4, 203, 137
    TX, TY = (W + 15) // 16, (H + 15) // 16
    S = 64  # 1/V of each tile's pixels per view: one image's worth over the batch
    pix = sample_lists(V, TX * TY, S, 5)
    v, y, x, inside = dense_index(pix, TX, H, W)
    dL_full = synth.make_dLdC_scaled(V, H, W, 7)
    dL_s = np.zeros(pix.shape + (3,), np.float32)
    dL_s[inside] = dL_full[v[inside], :, y[inside], x[inside]]
    dL_masked = np.zeros_like(dL_full)
    dL_masked[v[inside], :, y[inside], x[inside]] = dL_full[v[inside], :, y[inside], x[inside]]
    o = oracle.Oracle(g, cams)
    ref = o.backward(dL_masked)
    im = o.image()
    return dict(g=g, cams=cams, pix=pix, S=S, idx=(v, y, x, inside), dL_s=dL_s, dL_masked=dL_masked, ref=ref, im=im,
                im32=o.image32())


@pytest.mark.parametrize("mode", [0, 1])
def test_partial_forward_equals_full_render(scene, mode):
    out = run_partial(scene["g"], scene["cams"], scene["pix"], mode)
    v, y, x, inside = scene["idx"]
    im = scene["im"]
    np.testing.assert_array_equal(out["n_contrib"][inside], im["n_contrib"][v[inside], y[inside], x[inside]])
    ref_rgb = im["rgb"].transpose(0, 2, 3, 1)[v[inside], y[inside], x[inside]]
    assert np.max(np.abs(out["rgb"][inside] - ref_rgb)) <= 1e-5
    np.testing.assert_array_equal(out["rgb"][inside],
                                  scene["im32"]["rgb"].transpose(0, 2, 3, 1)[v[inside], y[inside], x[inside]])
    assert np.max(np.abs(out["T_final"][inside] - im["T_final"][v[inside], y[inside], x[inside]])) <= 1e-5
    assert np.all(out["n_contrib"][~inside] == 0) and np.all(out["T_final"][~inside] == 1.0)


def test_thread_efficient_and_masked_agree_bitwise(scene):
    a = run_partial(scene["g"], scene["cams"], scene["pix"], 0)
    b = run_partial(scene["g"], scene["cams"], scene["pix"], 1)
    for k in ("rgb", "T_final", "n_contrib"):
        np.testing.assert_array_equal(a[k], b[k])


@pytest.mark.parametrize("mode", [0, 1])
def test_partial_backward_equals_masked_full_backward(scene, mode):
    out = run_partial(scene["g"], scene["cams"], scene["pix"], mode, scene["dL_s"])
    ref = scene["ref"]
    scale = per_view_scale(scene["g"], scene["cams"], scene["dL_masked"])
    for k in ["d_means", "d_log_scales", "d_quats", "d_opacity_logits", "d_sh", "e1", "e2", "e_old"]:
        assert_close_rel(out[k], ref[k], k, scale=scale[k])
    np.testing.assert_array_equal(out["vis"], ref["vis"])


def test_identity_list_equals_full_kernel(scene):
    """S = 256 with every pixel listed reproduces the full render (GPU vs GPU, bit-exact counts)."""
    from gpu_harness import run_gpu
    V, T = scene["pix"].shape[:2]
    ident = np.tile(np.arange(256, dtype=np.int32), (V, T, 1))
    a = run_partial(scene["g"], scene["cams"], ident, 0)
    full = run_gpu(scene["g"], scene["cams"], None, export=False)
    v, y, x, inside = dense_index(ident, (203 + 15) // 16, 137, 203)
    np.testing.assert_array_equal(a["n_contrib"][inside], full["n_contrib"][v[inside], y[inside], x[inside]])
    assert np.max(np.abs(a["rgb"][inside] - full["rgb"].transpose(0, 2, 3, 1)[v[inside], y[inside], x[inside]])) <= 1e-6


def test_occupancy_counts(scene):
    """threads launched / holding a pixel, counted by the kernel.  Masked:
    256 threads per (view, tile), the listed in-image pixels active; thread-efficient:
    ⌈S/32⌉·32 threads, the same pixels active; lane-steps of the entry walk: efficient
    wastes no more than masked."""
    v, y, x, inside = scene["idx"]
    pix = scene["pix"]
    V, T, S = pix.shape
    n_in = int(np.count_nonzero(inside))
    occ = {m: run_partial(scene["g"], scene["cams"], pix, m)["occ"] for m in (0, 1)}
    eff, msk = occ[0], occ[1]  # mode 0: thread-efficient, 1: masked
    assert msk["threads_launched"] == V * T * 256
    assert eff["threads_launched"] == V * T * (-(-S // 32) * 32)
    assert msk["threads_active"] == n_in and eff["threads_active"] == n_in
    assert eff["lane_steps_active"] == msk["lane_steps_active"]  # the same pixels walk the same entries
    assert eff["lane_steps_active"] / eff["lane_steps_launched"] >= msk["lane_steps_active"] / msk["lane_steps_launched"]
