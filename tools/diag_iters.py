import math, sys, os, time
sys.path.insert(0, '.')
import numpy as np, synth
from paper_2511_17107_b200 import api
PI = math.pi
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
A = synth.lattice("fcc"); masks = synth.make_masks("fcc_diamond", A, n)
ctx = api.pc_create(A, n, synth.eps_pseudochiral(), masks)
kp = synth.kpath("fcc", 8)
for guard in (2, 3, 5, 8):
    api.pc_set_option(ctx, "guard", guard)
    its = []
    t = time.time()
    for g in (0, 10, 20, 30, 40):
        api.pc_set_option(ctx, "kindex_offset", g)
        r = api.pc_bands(ctx, kp[g:g+1], nev=10, tol=1e-5)
        its.append(int(r["iters"][0]))
    print("guard", guard, "iters", its, "mean", np.mean(its), "time/k", (time.time()-t)/5, flush=True)
api.pc_set_option(ctx, "guard", 5)
api.pc_set_option(ctx, "verbose", 1)
api.pc_set_option(ctx, "kindex_offset", 20)
r = api.pc_bands(ctx, kp[20:21], nev=10, tol=1e-5)
