import sys, math
sys.path.insert(0, "/root/repo")
import numpy as np, synth
from paper_2511_17107_b200 import api
PI = math.pi
for lat in ("sc", "fcc"):
    A = synth.lattice(lat)
    for d in (0, 1):
        ctx = api.pc_create(A, 8, synth.eps_pseudochiral(), synth.make_masks("full", A, 8))
        api.pc_set_option(ctx, "gram_derive", d)
        api.pc_set_option(ctx, "verbose", 1)
        r = api.pc_bands(ctx, [[PI, PI, PI]], nev=10, tol=1e-7, maxit=60)
        print(lat, d, r["status"], r["iters"], file=sys.stderr, flush=True)
        ctx.close()
