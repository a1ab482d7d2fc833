import math, sys, os, time
sys.path.insert(0, '.')
import numpy as np, synth
from paper_2511_17107_b200 import api
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
A = synth.lattice("fcc"); masks = synth.make_masks("fcc_diamond", A, n)
ctx = api.pc_create(A, n, synth.eps_pseudochiral(), masks)
kp = synth.kpath("fcc", 8)
ref = None
for start, noise in ((0, 0), (1, 1e-3), (1, 1e-1), (1, 0.0)):
    api.pc_set_option(ctx, "start", start); api.pc_set_option(ctx, "start_noise", noise)
    its, oms = [], []
    t = time.time()
    for g in (0, 10, 20, 24, 30, 40):
        api.pc_set_option(ctx, "kindex_offset", g)
        r = api.pc_bands(ctx, kp[g:g+1], nev=10, tol=1e-5)
        its.append(int(r["iters"][0])); oms.append(r["omega2"][0])
    oms = np.array(oms)
    if ref is None: ref = oms
    print("start", start, "noise", noise, "iters", its, "mean", np.mean(its), "time/k %.3f" % ((time.time()-t)/6),
          "max rel diff vs random start %.1e" % np.max(np.abs(oms-ref)/ref), flush=True)
vac = api.pc_create(np.eye(3), 8, np.eye(3), np.zeros((4, 8, 8, 8), np.uint8))
r = api.pc_bands(vac, [[math.pi]*3, [math.pi/7, 3*math.pi/5, 4*math.pi/13]], nev=6, tol=1e-7)
print("vacuum", r["iters"], r["status"], r["omega2"])
