"""Phase timing of the bench's end-to-end job (pc_create from pinned host masks, solve_concurrent,
pc_destroy) for option values, to locate overheads outside the kernels.

usage: python tools/e2e_probe.py [--key update_tmap --values 0 1] [--nk 4] [--ctx 2]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2511_17107_b200 import api, bands  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--key", default="update_tmap")
ap.add_argument("--values", type=float, nargs="+", default=[0, 1])
ap.add_argument("--nk", type=int, default=4)
ap.add_argument("--ctx", type=int, default=2)
ap.add_argument("--keep", type=int, default=1, help="long-lived contexts alive during the job (as in bench)")
a = ap.parse_args()
W = synth.WORKLOADS["C4"]
A = W.A()
masks = synth.make_masks(W.geometry, A, W.n)
pin = torch.from_numpy(masks.reshape(-1)).pin_memory().numpy().reshape(masks.shape)
kp = synth.kpath(W.lattice, W.segments)
keep = [api.pc_create(A, W.n, W.eps1(), masks) for _ in range(a.keep)]
for c in keep:
    bands.solve_local(c, kp, [1], W.nev, 1e-5, 5, 0)
for rep in range(2):
    for v in a.values:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ce = [api.pc_create(A, W.n, W.eps1(), pin) for _ in range(a.ctx)]
        for c in ce:
            api.pc_set_option(c, a.key, v)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        out = bands.solve_concurrent(ce, kp, list(range(1, 1 + a.nk)), W.nev, 1e-5, 1000, 0)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        for c in ce:
            c.close()
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        print(f"rep {rep} {a.key}={v}: create {t1 - t0:.3f}s solve {t2 - t1:.3f}s destroy {t3 - t2:.3f}s "
              f"iters {out[2].tolist()} kpts/s {a.nk / (t3 - t0):.3f}", flush=True)
