"""Verbose pc_bands on the n=128 FCC vacuum case of test_bands_vacuum_closed_form_large (diagnostics)."""
import math, sys
sys.path.insert(0, '.')
import numpy as np
import synth
from paper_2511_17107_b200 import api
PI = math.pi
n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
A = synth.lattice("fcc")
for d in (0, 1):
    ctx = api.pc_create(A, n, np.eye(3), np.zeros((4, n, n, n), np.uint8))
    api.pc_set_option(ctx, "verbose", 1)
    api.pc_set_option(ctx, "gram_derive", d)
    r = api.pc_bands(ctx, [[PI, PI, PI]], nev=10, tol=1e-6, maxit=60)
    print("derive", d, r["omega2"][0], r["iters"], r["status"], file=sys.stderr, flush=True)
    ctx.close()
