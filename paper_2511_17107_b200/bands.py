"""Band structure over a k-path, sharded across GPUs.

Bloch vectors are independent eigenproblems.  The k-points are handed out by a
dynamic queue (KQueue): one atomic counter in the process group's store (TCPStore.add) gives every
host thread of every rank the next position of a longest-first order of the k indices, so a rank
that drew cheap k-points takes more of them.  Each rank solves what it drew with pc_bands on its own
GPU (several concurrent contexts per GPU, one host thread each), and ONE collective gathers the
results (all_gather_into_tensor of padded per-rank blocks: k index, omega^2, Res_j, iterations,
status).  Start blocks are keyed by the global k index (pc_set_option "kindex_offset"), so the
eigenvalues do not depend on the number of GPUs or on which rank drew which k-point.

Static efficiency bound with a fixed partition: ceil(nk/G) k-points on the busiest of G ranks, e.g.
49 k-points on 8 GPUs -> 49 / (8 * 7) = 87.5 %.  With the queue the bound is set by the last k-point
to start: the makespan exceeds the mean load by at most one k-point's time, and longest-first order
(estimated costs, e.g. a previous run's iteration counts) makes that last item a short one.
"""
from __future__ import annotations

import threading
from typing import Callable

import numpy as np


def shard(nk: int, world: int, rank: int) -> list:
    """Global k indices owned by `rank` (round-robin)."""
    return list(range(rank, nk, world))


def shard_contiguous(nk: int, world: int, rank: int) -> list:
    """Global k indices owned by `rank` as one contiguous stretch of the path (warm-start mode:
    neighbouring k-points stay on one rank)."""
    base, extra = divmod(nk, world)
    lo = rank * base + min(rank, extra)
    return list(range(lo, lo + base + (1 if rank < extra else 0)))


def local_capacity(nk: int, world: int) -> int:
    return (nk + world - 1) // world


class KQueue:
    """Dynamic queue of global k indices shared by all ranks and all host threads of a rank.

    order: the k indices in hand-out order (see longest_first); store: a torch.distributed Store
    (its add() is atomic across processes) or None for a single process; key: counter name, unique
    per job (every rank must use the same key).  next() returns the next k index or None."""

    def __init__(self, order, store=None, key: str = "pcband/kq"):
        self.order = [int(g) for g in order]
        self.store = store
        self.key = key
        self._lock = threading.Lock()
        self._pos = 0

    def next(self):
        if self.store is not None:
            t = int(self.store.add(self.key, 1)) - 1
        else:
            with self._lock:
                t = self._pos
                self._pos += 1
        return self.order[t] if t < len(self.order) else None


class ChunkQueue(KQueue):
    """A KQueue whose items are chunks (lists) of k indices."""

    def __init__(self, chunks, store=None, key: str = "pcband/kq"):
        super().__init__(range(len(chunks)), store, key)
        self.chunks = [list(ch) for ch in chunks]

    def next(self):
        t = super().next()
        return None if t is None else self.chunks[t]


def longest_first(idx, cost=None) -> list:
    """Hand-out order: descending estimated cost (ties and cost=None: the given order)."""
    idx = [int(g) for g in idx]
    if cost is None:
        return idx
    c = np.asarray(cost, dtype=np.float64)
    return [g for _, g in sorted(((-c[g], t), g) for t, g in enumerate(idx))]


_JOBS = [0]


def job_queue(idx, cost=None, group=None, kbatch: int = 1) -> KQueue:
    """A KQueue over idx for this job: across ranks through the default process group's store
    (world > 1), else a local counter.  Collective in the sense that every rank must call it the
    same number of times (the counter key is numbered per call)."""
    import torch.distributed as dist
    order = longest_first(idx, cost)
    _JOBS[0] += 1
    store, key = None, "pcband/kq"
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        from torch.distributed import distributed_c10d as c10d
        store, key = c10d._get_default_store(), f"pcband/kq/{_JOBS[0]}"
    if kbatch > 1:  # chunks of consecutive path points (lock-step batches), in index order
        srt = sorted(int(g) for g in idx)
        return ChunkQueue([srt[i:i + kbatch] for i in range(0, len(srt), kbatch)], store, key)
    return KQueue(order, store, key)


def runs(ks):
    """Split a list of k indices into runs of consecutive integers (pc_bands keys the start block of its
    i-th k-point by kindex_offset + i)."""
    out = []
    for g in ks:
        if out and g == out[-1][-1] + 1:
            out[-1].append(g)
        else:
            out.append([g])
    return out


def solve_queue(ctxs, kpts: np.ndarray, queue: KQueue, nev: int, tol: float, maxit: int, seed: int,
                kbatch: int = 1):
    """Solve k-points drawn from `queue` with the contexts ctxs (one host thread per context; ctypes
    releases the GIL during pc_bands) until the queue is empty.  kbatch > 1: each draw hands out a chunk of
    kbatch k-points (queue items are chunk numbers of chunked(ks, kbatch)), solved in lock step by one
    pc_bands call per run of consecutive indices (option "kbatch").  Returns (idx, omega2, Res,
    iters, status) for the k-points this process solved, in the order they were drawn."""
    from . import api
    if not isinstance(ctxs, (list, tuple)):
        ctxs = [ctxs]
    rows = []
    lock = threading.Lock()
    errors = []

    def worker(ctx):
        try:
            if kbatch > 1:
                api.pc_set_option(ctx, "kbatch", kbatch)
            while True:
                item = queue.next()
                if item is None:
                    return
                for run in runs(item if isinstance(item, list) else [item]):
                    api.pc_set_option(ctx, "kindex_offset", run[0])
                    r = api.pc_bands(ctx, kpts[run], nev=nev, tol=tol, maxit=maxit, seed=seed)
                    with lock:
                        for t, g in enumerate(run):
                            rows.append((g, r["omega2"][t], r["resid"][t], int(r["iters"][t]), int(r["status"][t])))
        except Exception as ex:  # pragma: no cover - surfaced below
            errors.append(ex)

    if len(ctxs) == 1:
        worker(ctxs[0])
    else:
        threads = [threading.Thread(target=worker, args=(c,)) for c in ctxs]
        for th in threads:
            th.start()
        for th in threads:
            th.join()
    if errors:
        raise errors[0]
    idx = [r[0] for r in rows]
    om = np.array([r[1] for r in rows]).reshape(len(rows), nev)
    rs = np.array([r[2] for r in rows]).reshape(len(rows), nev)
    it = np.array([r[3] for r in rows], dtype=np.int64)
    stt = np.array([r[4] for r in rows], dtype=np.int64)
    return idx, om, rs, it, stt


def _in_order(idx, got):
    """Reorder solve_queue output (drawn order) to the order of idx."""
    g_idx, om, rs, it, stt = got
    pos = {g: t for t, g in enumerate(g_idx)}
    sel = [pos[g] for g in idx]
    return om[sel], rs[sel], it[sel], stt[sel]


def solve_local(ctx, kpts: np.ndarray, idx: list, nev: int, tol: float, maxit: int, seed: int):
    """Solve the k-points idx (in order) on one context; each start block is keyed by its global
    index.  Returns (omega2, Res, iters, status) in the order of idx."""
    return _in_order(idx, solve_queue([ctx], kpts, KQueue(idx), nev, tol, maxit, seed))


def solve_concurrent(ctxs, kpts: np.ndarray, idx: list, nev: int, tol: float, maxit: int, seed: int):
    """Solve the k-points idx with len(ctxs) independent contexts on one GPU, one host thread each
    (each context owns its CUDA stream and workspace), drawing from one local queue in index order, so
    the single-CTA Rayleigh-Ritz steps and host round trips of one k-point overlap the bulk kernels of
    another.  Results (in the order of idx) do not depend on the number of contexts."""
    return _in_order(idx, solve_queue(list(ctxs), kpts, KQueue(idx), nev, tol, maxit, seed))


def solve_warm(ctxs, kpts: np.ndarray, idx: list, nev: int, tol: float, maxit: int, seed: int):
    """Warm-started path continuation (not in the paper): idx is split into
    len(ctxs) contiguous stretches, each solved in path order on its own context with the option
    warm_start = 1 (the start block of k_i is the Ritz block of k_{i-1}; k = 0 exactly still starts
    cold).  Contexts run concurrently, one host thread each."""
    import threading
    from . import api
    om = np.zeros((len(idx), nev))
    rs = np.zeros((len(idx), nev))
    it = np.zeros(len(idx), dtype=np.int64)
    stt = np.zeros(len(idx), dtype=np.int64)
    parts = [shard_contiguous(len(idx), len(ctxs), r) for r in range(len(ctxs))]
    errors = []

    def worker(ctx, ts):
        try:
            api.pc_set_option(ctx, "warm_start", 1)
            for t in ts:
                g = idx[t]
                api.pc_set_option(ctx, "kindex_offset", g)
                r = api.pc_bands(ctx, kpts[g:g + 1], nev=nev, tol=tol, maxit=maxit, seed=seed)
                om[t], rs[t], it[t], stt[t] = r["omega2"][0], r["resid"][0], r["iters"][0], r["status"][0]
            api.pc_set_option(ctx, "warm_start", 0)
        except Exception as ex:  # pragma: no cover - surfaced below
            errors.append(ex)

    threads = [threading.Thread(target=worker, args=(c, ts)) for c, ts in zip(ctxs, parts)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    if errors:
        raise errors[0]
    return om, rs, it, stt


def gather(om, rs, it, stt, idx, nk, group=None, device=None, cap=None, ks=None):
    """All-gather the per-rank results (one collective) and scatter them into k order.  cap = rows per
    rank in the collective (default: the static round-robin share; with the dynamic queue a rank can
    hold up to all len(ks) k-points).  ks: the global indices that must be present (default all nk)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    nev = om.shape[1]
    if cap is None:
        cap = local_capacity(nk, world)
    # packed row per local k: [global index, omega2 (nev), resid (nev), iters, status]
    width = 2 * nev + 3
    buf = np.full((cap, width), -1.0)
    for t, g in enumerate(idx):
        buf[t, 0] = g
        buf[t, 1:1 + nev] = om[t]
        buf[t, 1 + nev:1 + 2 * nev] = rs[t]
        buf[t, 1 + 2 * nev] = it[t]
        buf[t, 2 + 2 * nev] = stt[t]
    local = torch.from_numpy(buf)
    if device is not None:
        local = local.to(device)
    if world > 1:
        out = torch.empty((world * cap, width), dtype=local.dtype, device=local.device)
        dist.all_gather_into_tensor(out, local, group=group)
    else:
        out = local
    allb = out.cpu().numpy()
    res = {"omega2": np.zeros((nk, nev)), "resid": np.zeros((nk, nev)),
           "iters": np.zeros(nk, dtype=np.int64), "status": np.zeros(nk, dtype=np.int64)}
    seen = np.zeros(nk, dtype=bool)
    for row in allb:
        g = int(row[0])
        if g < 0:
            continue
        res["omega2"][g] = row[1:1 + nev]
        res["resid"][g] = row[1 + nev:1 + 2 * nev]
        res["iters"][g] = int(row[1 + 2 * nev])
        res["status"][g] = int(row[2 + 2 * nev])
        seen[g] = True
    need = np.arange(nk) if ks is None else np.asarray(ks, dtype=np.int64)
    if not seen[need].all():
        raise RuntimeError("band gather lost k-points")
    return res


def band_structure(ctxs, kpts, nev=10, tol=1e-5, maxit=500, seed=0, group=None, device=None,
                   solver: Callable | None = None, cost=None, ks=None, kbatch: int = 1):
    """Full band structure through the public API: the k-points (all of kpts, or the global indices
    ks) are drawn from a dynamic queue shared by every rank (longest-first by `cost` if given), solved
    by this rank's contexts ctxs (one or a list: concurrent solves on one GPU), and gathered with one
    all-gather.  Every rank returns the full result in k order.  `solver(ctxs, kpts, queue, nev, tol,
    maxit, seed)` replaces solve_queue in host-logic tests (a CPU stub under gloo).  kbatch > 1: chunks of
    kbatch consecutive k-points are drawn and solved in lock step (option "kbatch"; n <= 64)."""
    kpts = np.asarray(kpts, dtype=np.float64).reshape(-1, 3)
    nk = kpts.shape[0]
    ks = list(range(nk)) if ks is None else [int(g) for g in ks]
    q = job_queue(ks, cost, group, kbatch)
    if solver is None:
        idx, om, rs, it, stt = solve_queue(ctxs, kpts, q, nev, tol, maxit, seed, kbatch)
    else:
        idx, om, rs, it, stt = solver(ctxs, kpts, q, nev, tol, maxit, seed)
    return gather(om, rs, it, stt, idx, nk, group=group, device=device, cap=len(ks), ks=ks)
