"""Host logic of the multi-GPU k-path sharding, world_size 2 over gloo on CPU.
The GPU solve is replaced by a deterministic stub keyed by the global k index -- this tests the
partition + single all-gather, not the numerics (those are the -m gpu tests)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2511_17107_b200 import bands


def stub_solver(ctx, kpts, idx, nev, tol, maxit, seed):
    om = np.array([[kpts[g].sum() + j + 0.25 * g for j in range(nev)] for g in idx]).reshape(len(idx), nev)
    rs = np.full((len(idx), nev), 1e-9)
    it = np.array([10 + g for g in idx], dtype=np.int64)
    st = np.zeros(len(idx), dtype=np.int64)
    return om, rs, it, st


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, nk, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    kp = np.arange(nk * 3, dtype=np.float64).reshape(nk, 3) * 0.1
    res = bands.band_structure(None, kp, nev=4, solver=stub_solver)
    if rank == 0:
        q.put({k: v.tolist() for k, v in res.items()})
    dist.destroy_process_group()


@pytest.mark.parametrize("nk,world", [(7, 2), (49, 2), (1, 2), (5, 3)])
def test_sharded_gather_matches_single(nk, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, nk, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    kp = np.arange(nk * 3, dtype=np.float64).reshape(nk, 3) * 0.1
    om, rs, it, st = stub_solver(None, kp, list(range(nk)), 4, 0, 0, 0)
    assert np.array_equal(np.array(got["omega2"]), om)
    assert np.array_equal(np.array(got["iters"]), it)


def test_shard_partition():
    for nk in (1, 7, 49, 193):
        for w in (1, 2, 4, 8):
            parts = [bands.shard(nk, w, r) for r in range(w)]
            flat = sorted(i for p in parts for i in p)
            assert flat == list(range(nk))
            assert max(len(p) for p in parts) == bands.local_capacity(nk, w)
