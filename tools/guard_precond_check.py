"""Block-size robustness check: pc_bands at several guard counts (block b = nev + guard), kernel
options and preconditioners against the default configuration's eigenvalues (FCC diamond
pseudochiral, n = 32, 4 k-points).  usage: python tools/guard_precond_check.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2511_17107_b200 import api  # noqa: E402

W = synth.WORKLOADS["C4"]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
A = W.A()
masks = synth.make_masks(W.geometry, A, n)
kp = synth.kpath(W.lattice, W.segments)[1:5]


def solve(opts, nev=10):
    ctx = api.pc_create(A, n, W.eps1(), masks)
    for k, v in opts.items():
        api.pc_set_option(ctx, k, v)
    try:
        r = api.pc_bands(ctx, kp, nev=nev, tol=1e-8, maxit=400)
        return r["omega2"], r["iters"].tolist(), r["status"].tolist()
    except Exception as e:  # noqa: BLE001
        return None, str(e), None
    finally:
        ctx.close()


ref, it0, st0 = solve({})
print("default", it0, st0, flush=True)
for nev in (10, 20):
    refn = ref if nev == 10 else solve({}, nev=20)[0]
    for g in ([1, 2, 3, 4, 5, 7, 8, 10] if nev == 10 else [5, 6]):
        for opts in ({"guard": g}, {"guard": g, "update_tmap": 0}, {"guard": g, "precond": 1}):
            om, it, st = solve(opts, nev)
            if om is None or refn is None:
                print(nev, opts, "ERR", it, flush=True)
            else:
                print(nev, opts, "iters", it, "status", st, "max rel diff", float(np.max(np.abs(om - refn) / refn)),
                      flush=True)
