"""N>1 path on CPU (gloo, world size 2): view sharding + the flat-buffer all-reduce
give the same gradients and E1/E2/vis as one process over all views.  The per-rank
compute here is the oracle (the GPU path needs a device); the layout, partition and
collective are the ones bench.py uses on NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2506_12727_b200.dist import GradBuffer, view_shard


def test_view_shard_partitions():
    for V in (1, 4, 7, 32):
        for W in (1, 2, 3, 8):
            spans = [view_shard(V, W, r) for r in range(W)]
            assert spans[0][0] == 0 and spans[-1][1] == V
            assert all(spans[i][1] == spans[i + 1][0] for i in range(W - 1))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import oracle
    import synth
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g, cams = synth.make_scene(synth.scaled(synth.CONFIGS["tiny"], P=300, V=5))
    dL = synth.make_dLdC_scaled(5, 64, 64, 3)
    lo, hi = view_shard(5, world, rank)
    o = oracle.Oracle(g, cams[lo:hi])
    r = o.backward(dL[lo:hi])
    r["gsum"] = o.adc_extra()["gsum"]
    buf = GradBuffer(300, 1, "cpu")
    for k, v in buf.views.items():
        v.copy_(torch.from_numpy(r[k].astype(np.float32)))
    buf.allreduce()
    buf.e_old.copy_(torch.linalg.norm(buf.views["gsum"], dim=1))  # (the library's E_old kernel on GPUs)
    if rank == 0:
        out = {k: v.numpy().copy() for k, v in buf.views.items()}
        out["e_old"] = buf.e_old.numpy().copy()
        q.put(out)
    dist.barrier()
    dist.destroy_process_group()


def _worker_chunked(rank, world, port, q):
    """The overlapped schedule: chunk-major buffer, per-chunk compute then async all-reduce."""
    import oracle
    import synth
    from paper_2506_12727_b200.dist import adc_stats_allreduce
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g, cams = synth.make_scene(synth.scaled(synth.CONFIGS["tiny"], P=700, V=5))
    dL = synth.make_dLdC_scaled(5, 64, 64, 3)
    lo, hi = view_shard(5, world, rank)
    o = oracle.Oracle(g, cams[lo:hi])
    r = o.backward(dL[lo:hi])
    r["gsum"] = o.adc_extra()["gsum"]
    buf = GradBuffer(700, 1, "cpu", chunks=3)
    assert len(buf.bounds) == 3 and all(a % 256 == 0 for a, _ in buf.bounds)
    seen = []

    def compute(c, a, b, gr, ad):  # what mvgs_adc_stats_range writes: rows a..b-1 at row 0
        seen.append(c)
        assert "e_old" not in ad  # per-rank E_old is not computed: it is not a sum over views
        for k, t in list(gr.items()) + [(k, ad[k]) for k in ("e1", "e2", "vis", "gsum")]:
            t.copy_(torch.from_numpy(r[k][a:b].astype(np.float32)))

    def e_old(c, a, b, gs, eo):  # what mvgs_e_old_from_gsum writes, after the chunk's sum
        eo.copy_(torch.linalg.norm(gs, dim=1))
    adc_stats_allreduce(None, buf, compute=compute, e_old=e_old)
    assert seen == [0, 1, 2]
    if rank == 0:
        out = {k: v.numpy().copy() for k, v in buf.views.items()}
        out["e_old"] = buf.e_old.numpy().copy()
        q.put(out)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("worker", ["plain", "chunked"])
def test_two_rank_allreduce_equals_single_process(worker):
    import oracle
    import synth
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    target = _worker if worker == "plain" else _worker_chunked
    P = 300 if worker == "plain" else 700
    procs = [ctx.Process(target=target, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g, cams = synth.make_scene(synth.scaled(synth.CONFIGS["tiny"], P=P, V=5))
    o = oracle.Oracle(g, cams)
    ref = o.backward(synth.make_dLdC_scaled(5, 64, 64, 3))
    ref["gsum"] = o.adc_extra()["gsum"]
    assert "e_old" in got  # the all-views E_old, from the summed gsum (R49)
    for k in got:
        np.testing.assert_allclose(got[k], ref[k].astype(np.float32), rtol=1e-5, atol=1e-6 * np.abs(ref[k]).max(),
                                   err_msg=k)


# ------------------------------------------------------------ owner-sharded exchange (lever 3)
def _synthetic_layout(V, P, seed=7):
    """Per-(view, 256-block) participation counts and the slot values a single GPU would hold:
    slot k of block b of view v carries the value v·1e6 + b·1e3 + k in all 12 floats."""
    rng = np.random.default_rng(seed)
    NB = -(-P // 256)
    cnt = rng.integers(0, 40, (V, NB))
    return cnt, NB


def _slots_of(cnt, views, blocks):
    vals = [np.full((int(cnt[v, b]), 12), v * 1e6 + b * 1e3, np.float32) + np.arange(int(cnt[v, b]), dtype=np.float32)[:, None]
            for v in views for b in blocks]
    return np.concatenate(vals) if vals else np.zeros((0, 12), np.float32)


def _worker_owner(rank, world, port, q):
    from paper_2506_12727_b200.dist import (check_plan_sizes, exchange_plan, owner_bounds, run_exchange,
                                            view_renderer)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    V, P = 7, 1900
    cnt, NB = _synthetic_layout(V, P)
    bounds = owner_bounds(P, world)
    ob = [(int(bounds[o]) // 256, -(-int(bounds[o + 1]) // 256)) for o in range(world)]
    renderer = view_renderer(V, world)
    mine = [v for v in range(V) if renderer[v] == rank]
    # this rank's slots: its views, view-major, blocks ascending (what mvgs_owner_slices describes)
    slots = torch.from_numpy(_slots_of(cnt, mine, range(NB)).reshape(-1))
    slot_off = np.zeros((len(mine), world + 1), np.int64)
    base = 0
    for l, v in enumerate(mine):
        for o in range(world):
            slot_off[l, o] = base + cnt[v, :ob[o][0]].sum()
        slot_off[l, world] = base + cnt[v].sum()
        base += cnt[v].sum()
    # the owner's layout: every view, its blocks only (what mvgs_owner_prepare describes)
    b0, b1 = ob[rank]
    view_off = np.concatenate([[0], np.cumsum([cnt[v, b0:b1].sum() for v in range(V)])]).astype(np.int64)
    recv = torch.full((int(view_off[-1]) * 12,), -1.0)
    check_plan_sizes(rank, world, renderer, slot_off, view_off, "cpu")
    run_exchange(exchange_plan(rank, world, renderer, slot_off, view_off), slots, recv)
    want = _slots_of(cnt, range(V), range(b0, b1)).reshape(-1)
    q.put((rank, bool(np.array_equal(recv.numpy(), want))))
    # a renderer whose slice disagrees with the owner's layout is caught before any transfer
    bad = slot_off.copy()
    if len(mine):
        bad[0, 1:] += 1
    try:
        check_plan_sizes(rank, world, renderer, bad, view_off, "cpu")
        q.put((rank, "mismatch not detected"))
    except RuntimeError:
        q.put((rank, "detected"))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_owner_exchange_delivers_the_single_gpu_layout(world):
    """Every owner receives exactly the slots a single GPU holding all views would have for its
    Gaussians, in its own view-major layout, through one batch of point-to-point transfers."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_owner, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2 * world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert sorted(r for r in res if r[1] is True) == [(r, True) for r in range(world)]
    assert sorted(r for r in res if r[1] == "detected") == [(r, "detected") for r in range(world)]


def test_owner_bounds():
    from paper_2506_12727_b200.dist import owner_bounds
    for P in (0, 1, 255, 256, 700, 5_000_000):
        for W in (1, 2, 3, 8):
            b = owner_bounds(P, W)
            assert b[0] == 0 and b[-1] == P and np.all(np.diff(b) >= 0) and len(b) == W + 1
            assert np.all((b[:-1] % 256 == 0) | (b[:-1] == P))  # an empty trailing range starts at P
