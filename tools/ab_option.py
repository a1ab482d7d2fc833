"""A/B a pc_set_option on the bench workload: per-class CUDA-event times and k-point throughput.

usage: python tools/ab_option.py --key fuse_resid --values 0 1 [--workload C4] [--nk 2]
"""
import argparse
import json
import math
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
ap.add_argument("--key", required=True)
ap.add_argument("--values", type=float, nargs="+", required=True)
ap.add_argument("--nk", type=int, default=2)
ap.add_argument("--tol", type=float, default=1e-5)
ap.add_argument("--maxit", type=int, default=1000)
ap.add_argument("--set", nargs="*", default=[], help="fixed options key=value applied first")
a = ap.parse_args()
W = synth.WORKLOADS[a.workload]
A = W.A()
masks = synth.make_masks(W.geometry, A, W.n)
kp = synth.kpath(W.lattice, W.segments)[1: 1 + a.nk]
ctx = api.pc_create(A, W.n, W.eps1(), masks)
for kv in a.set:
    api.pc_set_option(ctx, kv.split("=")[0], float(kv.split("=")[1]))
api.pc_bands(ctx, kp[:1], nev=W.nev, tol=a.tol, maxit=20)  # warm-up
out = {}
for v in a.values:
    api.pc_set_option(ctx, a.key, v)
    api.pc_set_option(ctx, "profile", 1)
    api.pc_stats(ctx, reset=True)
    torch.cuda.synchronize()
    t = time.time()
    r = api.pc_bands(ctx, kp, nev=W.nev, tol=a.tol, maxit=a.maxit)
    torch.cuda.synchronize()
    el = time.time() - t
    st = api.pc_stats(ctx)
    its = int(r["iters"].sum())
    row = {"seconds": el, "kpts_per_s": len(kp) / el, "iters": r["iters"].tolist(),
           "ms_per_it": 1e3 * el / max(its, 1), "launches": st.pop("launches"),
           "omega2_k0": r["omega2"][0][:4].tolist(), "resid_max": float(r["resid"].max()),
           "class_ms_per_it": {k: round(s["ms"] / max(its, 1), 4) for k, s in st.items() if s["count"]}}
    out[str(v)] = row
    print(a.key, v, json.dumps(row), flush=True)
