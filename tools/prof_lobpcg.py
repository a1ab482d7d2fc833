"""Short LOBPCG run at the bench workload for ncu captures: one k-point, a few iterations."""
import argparse, math, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2511_17107_b200 import api
ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="C4")
ap.add_argument("--maxit", type=int, default=3)
ap.add_argument("--n", type=int, default=0)
a = ap.parse_args()
W = synth.WORKLOADS[a.workload]
n = a.n or W.n
A = W.A()
masks = synth.make_masks(W.geometry, A, n)
ctx = api.pc_create(A, n, W.eps1(), masks)
r = api.pc_bands(ctx, [[math.pi, math.pi, math.pi]], nev=W.nev, tol=1e-5, maxit=a.maxit)
torch.cuda.synchronize()
print("iters", r["iters"], "omega2", r["omega2"][0][:3])
