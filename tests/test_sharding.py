"""Host logic of the multi-GPU k-path distribution over gloo on CPU, world sizes 2 and 4:
the dynamic queue (one atomic counter in the process group's store), the single all-gather, and the
longest-first order.  The GPU solve is replaced by a deterministic stub keyed by the global k index --
this tests the distribution, not the numerics (those are the -m gpu tests)."""
import os
import socket
import time

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2511_17107_b200 import bands


def stub_values(kpts, g, nev):
    return np.array([kpts[g].sum() + j + 0.25 * g for j in range(nev)])


def stub_solver(ctxs, kpts, queue, nev, tol, maxit, seed):
    """Draws from the shared queue like bands.solve_queue; k-point g 'costs' (g % 3) ms."""
    rows = []
    while True:
        g = queue.next()
        if g is None:
            break
        time.sleep(0.001 * (g % 3))
        rows.append(g)
    om = np.array([stub_values(kpts, g, nev) for g in rows]).reshape(len(rows), nev)
    rs = np.full((len(rows), nev), 1e-9)
    it = np.array([10 + g for g in rows], dtype=np.int64)
    st = np.zeros(len(rows), dtype=np.int64)
    return rows, om, rs, it, st


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, nk, q, jobs):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    kp = np.arange(nk * 3, dtype=np.float64).reshape(nk, 3) * 0.1
    drawn = []

    def counting_solver(*a):
        out = stub_solver(*a)
        drawn.append(list(out[0]))
        return out

    results = []
    for j in range(jobs):  # several jobs in a row: each gets its own counter
        cost = np.arange(nk)[::-1] if j % 2 else None
        res = bands.band_structure(None, kp, nev=4, solver=counting_solver, cost=cost)
        results.append({k: v.tolist() for k, v in res.items()})
    q.put((rank, drawn, results))
    dist.destroy_process_group()


@pytest.mark.parametrize("nk,world", [(7, 2), (49, 2), (1, 2), (5, 4), (49, 4)])
def test_queue_gather_matches_single(nk, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    jobs = 2
    procs = [ctx.Process(target=_worker, args=(r, world, port, nk, q, jobs)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    kp = np.arange(nk * 3, dtype=np.float64).reshape(nk, 3) * 0.1
    ref = np.array([stub_values(kp, g, 4) for g in range(nk)])
    for j in range(jobs):
        # every k-point solved exactly once across all ranks (dynamic queue, no duplicates)
        allk = sorted(g for _, drawn, _ in got for g in drawn[j])
        assert allk == list(range(nk))
        for _, _, results in got:  # every rank returns the full, k-ordered result
            assert np.array_equal(np.array(results[j]["omega2"]), ref)
            assert np.array_equal(np.array(results[j]["iters"]), 10 + np.arange(nk))


def test_queue_single_process_threads():
    """Without a process group the queue is a local counter shared by host threads."""
    import threading
    q = bands.KQueue(range(100))
    seen = []
    lock = threading.Lock()

    def w():
        while True:
            g = q.next()
            if g is None:
                return
            with lock:
                seen.append(g)

    th = [threading.Thread(target=w) for _ in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert sorted(seen) == list(range(100))


def test_longest_first_order():
    cost = np.array([5, 1, 9, 9, 3])
    assert bands.longest_first([0, 1, 2, 3, 4], cost) == [2, 3, 0, 4, 1]
    assert bands.longest_first([4, 1, 0]) == [4, 1, 0]


def test_shard_partition():
    for nk in (1, 7, 49, 193):
        for w in (1, 2, 4, 8):
            parts = [bands.shard(nk, w, r) for r in range(w)]
            flat = sorted(i for p in parts for i in p)
            assert flat == list(range(nk))
            assert max(len(p) for p in parts) == bands.local_capacity(nk, w)


def test_chunk_queue_and_runs():
    """kbatch > 1: the queue hands out chunks of consecutive k indices (lock-step batches); a chunk with a
    gap is split into runs of consecutive indices (pc_bands keys start blocks by kindex_offset + i)."""
    q = bands.job_queue([9, 3, 4, 5, 6, 0, 1, 2], kbatch=3)
    got = []
    while True:
        ch = q.next()
        if ch is None:
            break
        got.append(ch)
    assert got == [[0, 1, 2], [3, 4, 5], [6, 9]]
    assert bands.runs([6, 9]) == [[6], [9]]
    assert bands.runs([3, 4, 5, 7, 8]) == [[3, 4, 5], [7, 8]]
