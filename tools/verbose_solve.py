import sys, os
sys.path.insert(0, '/root/repo')
import numpy as np, synth
from paper_2511_17107_b200 import api
n = int(sys.argv[1]); wg = int(sys.argv[2])
A = synth.lattice("fcc"); masks = synth.make_masks("fcc_diamond", A, n)
eps1 = synth.eps_pseudochiral(13.0, 0.875)
kp = synth.kpath("fcc", 8)
ctx = api.pc_create(A, n, eps1, masks)
api.pc_set_option(ctx, "w_guard", wg)
api.pc_set_option(ctx, "verbose", 1)
r = api.pc_bands(ctx, kp[24:25], nev=10, tol=1e-5, maxit=1000)
print("iters", r["iters"], file=sys.stderr)
