"""Band structure over a k-path, sharded across GPUs.

Bloch vectors are independent eigenproblems: each rank owns a subset of the
k-points (round-robin, so neighbouring -- similarly expensive -- k-points spread across ranks),
solves them with pc_bands on its own GPU, and ONE collective gathers the results
(all_gather_into_tensor of padded per-rank blocks: omega^2, Res_j, iterations, status).  Start
blocks are keyed by the global k index (pc_set_option "kindex_offset"), so the eigenvalues do not
depend on the number of GPUs.
"""
from __future__ import annotations

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


def solve_local(ctx, kpts: np.ndarray, idx: list, nev: int, tol: float, maxit: int, seed: int):
    """Solve the k-points idx on this rank's context; per-k call so each start block is keyed by
    its global index."""
    from . import api
    om = np.zeros((len(idx), nev))
    rs = np.zeros((len(idx), nev))
    it = np.zeros(len(idx), dtype=np.int64)
    stt = np.zeros(len(idx), dtype=np.int64)
    for t, g in enumerate(idx):
        api.pc_set_option(ctx, "kindex_offset", g)
        r = api.pc_bands(ctx, kpts[g:g + 1], nev=nev, tol=tol, maxit=maxit, seed=seed)
        om[t], rs[t], it[t], stt[t] = r["omega2"][0], r["resid"][0], r["iters"][0], r["status"][0]
    return om, rs, it, stt


def solve_concurrent(ctxs, kpts: np.ndarray, idx: list, nev: int, tol: float, maxit: int, seed: int):
    """Solve the k-points idx with len(ctxs) independent contexts on one GPU, one host thread each
    (each context owns its CUDA stream and workspace; ctypes releases the GIL during pc_bands), so
    the single-CTA Rayleigh-Ritz steps and host round trips of one k-point overlap the bulk kernels
    of another.  Work is handed out from a shared queue in index order; results are independent of
    the number of contexts (start blocks are keyed by the global k index)."""
    import threading
    from . import api
    om = np.zeros((len(idx), nev))
    rs = np.zeros((len(idx), nev))
    it = np.zeros(len(idx), dtype=np.int64)
    stt = np.zeros(len(idx), dtype=np.int64)
    lock = threading.Lock()
    nxt = [0]
    errors = []

    def worker(ctx):
        try:
            while True:
                with lock:
                    t = nxt[0]
                    nxt[0] += 1
                if t >= len(idx):
                    return
                g = idx[t]
                api.pc_set_option(ctx, "kindex_offset", g)
                r = api.pc_bands(ctx, kpts[g:g + 1], nev=nev, tol=tol, maxit=maxit, seed=seed)
                om[t], rs[t], it[t], stt[t] = r["omega2"][0], r["resid"][0], r["iters"][0], r["status"][0]
        except Exception as ex:  # pragma: no cover - surfaced below
            errors.append(ex)

    threads = [threading.Thread(target=worker, args=(c,)) for c in ctxs]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    if errors:
        raise errors[0]
    return om, rs, it, stt


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


def gather(om, rs, it, stt, idx, nk, group=None, device=None):
    """All-gather the per-rank results (one collective) and scatter them into k order."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    nev = om.shape[1]
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
    if not seen.all():
        raise RuntimeError("band gather lost k-points")
    return res


def band_structure(ctx, kpts, nev=10, tol=1e-5, maxit=500, seed=0, group=None, device=None,
                   solver: Callable | None = None):
    """Full band structure: shard, solve locally (GPU), gather.  `solver` replaces solve_local in
    host-logic tests (e.g. a CPU stub under gloo)."""
    import torch.distributed as dist
    kpts = np.asarray(kpts, dtype=np.float64).reshape(-1, 3)
    nk = kpts.shape[0]
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    idx = shard(nk, world, rank)
    fn = solver or solve_local
    om, rs, it, stt = fn(ctx, kpts, idx, nev, tol, maxit, seed)
    return gather(om, rs, it, stt, idx, nk, group=group, device=device)
