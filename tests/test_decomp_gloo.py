"""Slab decomposition exchange on world_size 2 and 3 over gloo (CPU): after
the exchange every rank's axis-0 ghost planes hold the periodic images of the
global array, exactly as the single-process wrap (mesh.py:118-139) would."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import numpy_oracle as npo


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n0, n1, n2, h, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1610_09146_b200 as fd
        rng = np.random.default_rng(0)
        glob = rng.standard_normal((3, n0 + 2 * h, n1 + 2 * h, n2 + 2 * h))
        want = npo.halo_exchange(glob.copy(), h)
        slab = fd.Slab.from_process_group(n0)
        lo, n = slab.offset0, slab.local_n0
        local = np.zeros((3, n + 2 * h, n1 + 2 * h, n2 + 2 * h))
        local[:, h:h + n] = want[:, h + lo:h + lo + n]   # interior planes
        t = torch.from_numpy(local)
        slab.exchange(t, h)
        got = t.numpy()
        ok = np.array_equal(got, want[:, lo:lo + n + 2 * h])
        # the per-stage exchange sends only the first nf fields (the five
        # conservative ones of a state): the others' ghosts stay untouched
        part = np.zeros_like(local)
        part[:, h:h + n] = want[:, h + lo:h + lo + n]
        tp = torch.from_numpy(part)
        slab.exchange(tp, h, nf=2)
        ok = ok and np.array_equal(tp.numpy()[:2], want[:2, lo:lo + n + 2 * h])
        ok = ok and not tp.numpy()[2, :h].any() and not tp.numpy()[2, n + h:].any()
        # allreduce helper
        s = slab.allreduce_sum(torch.tensor([float(rank + 1)]))
        q.put((rank, ok, float(s[0])))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n0", [(2, 8), (3, 10), (4, 9)])
def test_slab_exchange_matches_periodic_wrap(world, n0):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n0, 5, 6, 2, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok, _ in res)
    assert all(s == world * (world + 1) / 2 for _, _, s in res)
