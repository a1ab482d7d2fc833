"""Sweep the LOBPCG block shape on one workload: guard columns (b = nev + guard) and how many of them
receive a search direction (w_guard; -1 = all).  Reports iterations and seconds per k-point on one
context (reading R14: block size and guard policy are not stated by the paper).

usage: python tools/guard_sweep.py [--workload C4] [--kidx 4 20 36] [--pairs 5,0 8,-1 ...]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2511_17107_b200 import api  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="C4")
ap.add_argument("--kidx", type=int, nargs="+", default=[4, 20, 36])
ap.add_argument("--pairs", nargs="+", default=["5,0", "5,2", "5,-1", "8,-1", "10,-1", "10,3", "10,5", "15,-1"])
ap.add_argument("--tol", type=float, default=1e-5)
ap.add_argument("--opts", nargs="*", default=[], help="extra key=value options")
a = ap.parse_args()
W = synth.WORKLOADS[a.workload]
A = W.A()
masks = synth.make_masks(W.geometry, A, W.n)
kp_all = synth.kpath(W.lattice, W.segments)
kp = kp_all[a.kidx]
ctx = api.pc_create(A, W.n, W.eps1(), masks)
for kv in a.opts:
    k, v = kv.split("=")
    api.pc_set_option(ctx, k, float(v))
api.pc_bands(ctx, kp[:1], nev=W.nev, tol=a.tol, maxit=10)  # warm-up
for pr in a.pairs:
    g, wg = (int(s) for s in pr.split(","))
    api.pc_set_option(ctx, "guard", g)
    api.pc_set_option(ctx, "w_guard", wg)
    its, secs, w0 = [], [], None
    for i, kk in zip(a.kidx, kp):
        api.pc_set_option(ctx, "kindex_offset", i)
        torch.cuda.synchronize()
        t = time.time()
        r = api.pc_bands(ctx, kk[None, :], nev=W.nev, tol=a.tol, maxit=1000)
        torch.cuda.synchronize()
        secs.append(time.time() - t)
        its.append(int(r["iters"][0]))
        if w0 is None:
            w0 = r["omega2"][0].tolist()
    row = {"guard": g, "w_guard": wg, "iters": its, "s_per_k": float(np.mean(secs)),
           "ms_per_it": 1e3 * float(np.sum(secs)) / max(1, sum(its)), "omega2_k0_last": w0[-1]}
    print(json.dumps(row), flush=True)
