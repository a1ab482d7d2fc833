import math, sys, time, numpy as np
sys.path.insert(0, '.')
import synth
from oracle import pc_oracle as O
from paper_2511_17107_b200 import api
PI = math.pi
cases = [("vac8", np.eye(3), np.eye(3), np.zeros((4,8,8,8),np.uint8), 8, (PI,PI,PI), 6),
         ("fcc8", synth.lattice("fcc"), synth.eps_pseudochiral(), synth.make_masks("random", synth.lattice("fcc"), 8, seed=3), 8, (0.7,-1.1,2.0), 10),
         ("fcc16", synth.lattice("fcc"), synth.eps_pseudochiral(), synth.make_masks("fcc_diamond", synth.lattice("fcc"), 16), 16, (PI,PI,PI), 10),
         ("sc32", np.eye(3), synth.eps_pseudochiral(), synth.make_masks("sc_curv", np.eye(3), 32), 32, (PI,PI,PI), 10)]
for dt in (1e-12, 1e-10, 1e-8):
    for tol in (1e-5, 1e-7, 1e-9):
        out = []
        for name, A, e, m, n, k, nev in cases:
            ctx = api.pc_create(A, n, e, m)
            api.pc_set_option(ctx, "drop_tol", dt)
            t = time.time()
            r = api.pc_bands(ctx, [k], nev=nev, tol=tol, maxit=300)
            out.append(f"{name}:it{r['iters'][0]}{'' if r['status'][0]==0 else 'X'}")
        print(f"drop {dt:.0e} tol {tol:.0e} ", " ".join(out), flush=True)
