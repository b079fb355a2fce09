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
    r = oracle.Oracle(g, cams[lo:hi]).backward(dL[lo:hi])
    buf = GradBuffer(300, 1, "cpu")
    for k, v in buf.views.items():
        v.copy_(torch.from_numpy(r[k].astype(np.float32)))
    buf.allreduce()
    if rank == 0:
        q.put({k: v.numpy().copy() for k, v in buf.views.items()})
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
    r = oracle.Oracle(g, cams[lo:hi]).backward(dL[lo:hi])
    buf = GradBuffer(700, 1, "cpu", chunks=3)
    assert len(buf.bounds) == 3 and all(a % 256 == 0 for a, _ in buf.bounds)
    seen = []

    def compute(c, a, b, gr, ad):  # what mvgs_adc_stats_range writes: rows a..b-1 at row 0
        seen.append(c)
        for k, t in list(gr.items()) + [(k, ad[k]) for k in ("e1", "e2", "vis")]:
            t.copy_(torch.from_numpy(r[k][a:b].astype(np.float32)))
    adc_stats_allreduce(None, buf, compute=compute)
    assert seen == [0, 1, 2]
    if rank == 0:
        q.put({k: v.numpy().copy() for k, v in buf.views.items()})
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
    ref = oracle.Oracle(g, cams).backward(synth.make_dLdC_scaled(5, 64, 64, 3))
    for k in got:
        np.testing.assert_allclose(got[k], ref[k].astype(np.float32), rtol=1e-5, atol=1e-6 * np.abs(ref[k]).max(),
                                   err_msg=k)
