"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck): every hot kernel family
at n = 8 and n = 32 (FFT passes, fused xex pass, K_P^{-1}, residual, Gram, TMA block update,
Rayleigh-Ritz) and the cluster plane pass at n = 128 (one column).

usage: compute-sanitizer --tool memcheck python tools/sanitize_run.py [--quick]
"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2511_17107_b200 import api  # noqa: E402

PI = math.pi


def run(n, nev, maxit, plane=False):
    A = synth.lattice("fcc")
    e = synth.eps_pseudochiral()
    masks = synth.make_masks("fcc_diamond", A, n)
    ctx = api.pc_create(A, n, e, masks)
    k = [PI, PI, PI]
    X = torch.from_numpy(synth.random_block(n, 3, seed=5)).cuda()
    Y = torch.empty_like(X)
    if plane:
        api.pc_set_option(ctx, "plane_fuse", 1)
        api.pc_apply(ctx, k, X[:1], Y[:1])
        torch.cuda.synchronize()
        print(f"n={n} plane pass ok", flush=True)
        return
    api.pc_apply(ctx, k, X, Y)
    api.pc_precond(ctx, k, X, Y)
    api.pc_fft3(ctx, X, Y)
    torch.cuda.synchronize()
    for opts in ({}, {"update_tmap": 0}, {"precond": 1}):
        for key, v in opts.items():
            api.pc_set_option(ctx, key, v)
        r = api.pc_bands(ctx, [k, [0.3, 0.2, 0.1]], nev=nev, tol=1e-6, maxit=maxit)
        print(f"n={n} {opts} iters {r['iters'].tolist()} w0 {r['omega2'][0][:3]}", flush=True)
        for key in opts:
            api.pc_set_option(ctx, key, {"update_tmap": 1, "precond": 0}[key])
    ctx.close()


if __name__ == "__main__":
    quick = "--quick" in sys.argv
    run(8, 6, 40)
    run(32, 10, 4 if quick else 12)
    if "--plane" in sys.argv:
        run(128, 10, 0, plane=True)
    print("sanitize workload done")
