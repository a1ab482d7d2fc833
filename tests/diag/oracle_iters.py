"""SciPy LOBPCG iteration count of the CPU oracle on a workload k-point (test infrastructure: imports
oracle/ and synth/ only).  Used by bench.py's cpu_baseline leg as the oracle's OWN iteration count
(not the paper's, not the GPU's) when it extrapolates a per-iteration timing to a k-point.

usage: python tests/diag/oracle_iters.py C4 5 [--tol 1e-5] [--out profiles/oracle_iters_c4.json]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from oracle import pc_oracle as O  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("workload")
ap.add_argument("kidx", type=int, nargs="+")
ap.add_argument("--tol", type=float, default=1e-5)
ap.add_argument("--out", default=None)
ap.add_argument("--n", type=int, default=0, help="grid size override (same lattice, geometry, eps1, path)")
a = ap.parse_args()
W = synth.WORKLOADS[a.workload]
if a.n:
    import dataclasses
    W = dataclasses.replace(W, n=a.n)
rows = []
for ki in a.kidx:
    k = W.kpoints()[ki]
    t0 = time.time()
    op = O.PenalizedOperator(W.n, k, W.A(), W.eps1(), W.masks(), "crossdof")
    info = {}
    ev, res = O.eigs_iterative(op, W.nev, tol=a.tol, seed=1000 + ki, maxiter=600, guard=5, info=info)
    rows.append({"kidx": ki, "k": k.tolist(), "tol": a.tol, "guard": 5, "iterations": info["iterations"],
                 "seconds": time.time() - t0, "omega2": ev.tolist(), "max_res": float(res.max())})
    print(json.dumps(rows[-1]), flush=True)
out = {"workload": a.workload, "n": W.n, "grid_override": bool(a.n), "nev": W.nev, "solver": "oracle eigs_iterative (SciPy LOBPCG, oracle K_P^-1)",
       "threads": os.environ.get("OMP_NUM_THREADS"), "rows": rows}
if a.out:
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
