"""k-point throughput of concurrent solves (bands.solve_concurrent) vs the number of contexts per GPU,
on the bench workload.

usage: python tools/conc_sweep.py [--nk 6] [--streams 2 3] [--opt key value ...]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2511_17107_b200 import api, bands  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="C4")
ap.add_argument("--nk", type=int, default=6)
ap.add_argument("--streams", type=int, nargs="+", default=[2, 3])
ap.add_argument("--opt", nargs=2, action="append", default=[], help="extra pc_set_option key value")
a = ap.parse_args()
W = synth.WORKLOADS[a.workload]
A = W.A()
masks = synth.make_masks(W.geometry, A, W.n)
kp = synth.kpath(W.lattice, W.segments)
idx = list(range(1, 1 + a.nk))
ctxs = [api.pc_create(A, W.n, W.eps1(), masks) for _ in range(max(a.streams))]
for c in ctxs:
    for k, v in a.opt:
        api.pc_set_option(c, k, float(v))
bands.solve_concurrent(ctxs[:2], kp, [0, 0], W.nev, 1e-5, 15, 0)  # warm-up (workspaces, JIT)
for s in a.streams:
    torch.cuda.synchronize()
    t = time.time()
    om, rs, it, st = bands.solve_concurrent(ctxs[:s], kp, idx, W.nev, 1e-5, 1000, 0)
    torch.cuda.synchronize()
    el = time.time() - t
    print(json.dumps({"streams": s, "kpts_per_s": len(idx) / el, "iters": it.tolist()}), flush=True)
