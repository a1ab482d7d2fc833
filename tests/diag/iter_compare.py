"""LOBPCG iteration counts: SciPy's LOBPCG (oracle operator + oracle K_P^{-1}) vs pc_bands option
variants, same operator, same k-points (Table 2 at P:1187-1203 for context).

usage: python tests/diag/iter_compare.py [--n 32] [--nk 4] [--which scipy,gpu] [--variants ...]
"""
import argparse
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import scipy.sparse.linalg as spla  # noqa: E402

import synth  # noqa: E402

VARIANTS = {
    "default": {},
    "wguard_all": {"w_guard": -1},
    "guard0": {"guard": 0},
    "guard3": {"guard": 3},
    "fullgram": {"gram_refresh": 1},
    "randstart": {"start": 0},
    "sticky": {"sticky_lock": 1},
}


def scipy_iters(n, A, eps1, masks, k, nev, guard, tol, seed=0):
    from oracle import pc_oracle as po
    op = po.PenalizedOperator(n, k, A, eps1, masks, "crossdof")

    def mv(X):
        X = np.asarray(X)
        return op.apply_fourier(X.T).T if X.ndim == 2 else op.apply_fourier(X[None, :])[0]

    def pc(X):
        X = np.asarray(X)
        if X.ndim == 1:
            return po.precond_fourier(n, op.k, op.A, op.gamma, X[None, :])[0]
        return po.precond_fourier(n, op.k, op.A, op.gamma, X.T).T

    dim = op.dim
    Aop = spla.LinearOperator((dim, dim), matvec=mv, matmat=mv, dtype=np.complex128)
    Mop = spla.LinearOperator((dim, dim), matvec=pc, matmat=pc, dtype=np.complex128)
    rng = np.random.default_rng(seed)
    m = nev + guard
    X0 = rng.standard_normal((dim, m)) + 1j * rng.standard_normal((dim, m))
    # stop on the first nev only: run with tol and check which columns count (SciPy checks all m)
    w, V, lh, rh = spla.lobpcg(Aop, X0, M=Mop, tol=tol, maxiter=1000, largest=False,
                               retLambdaHistory=True, retResidualNormsHistory=True)
    rh = np.array([np.asarray(r)[:m] for r in rh])
    # first iteration where the nev smallest Ritz pairs are all below tol
    its = None
    for i, (lam, r) in enumerate(zip(lh, rh)):
        o = np.argsort(lam)[:nev]
        if np.all(r[o] <= tol):
            its = i
            break
    return its, len(rh), np.sort(w)[:nev]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=32)
    ap.add_argument("--nk", type=int, default=4)
    ap.add_argument("--which", default="scipy,gpu")
    ap.add_argument("--variants", default=",".join(VARIANTS))
    ap.add_argument("--geometry", default="fcc_diamond")
    ap.add_argument("--lattice", default="fcc")
    ap.add_argument("--eps", default="pc13")
    ap.add_argument("--tol", type=float, default=1e-5)
    a = ap.parse_args()
    nev = 10
    A = synth.lattice(a.lattice)
    masks = synth.make_masks(a.geometry, A, a.n)
    eps1 = synth.eps_pseudochiral(13.0, 0.875) if a.eps == "pc13" else synth.eps_isotropic(13.0)
    kp = synth.kpath(a.lattice, 8)
    sel = np.linspace(1, len(kp) - 1, a.nk).astype(int)
    ks = kp[sel]
    out = {"n": a.n, "k_index": sel.tolist(), "scipy": {}, "gpu": {}}
    if "scipy" in a.which:
        for g in (0, 5):
            its, tot, w = [], [], None
            t = time.time()
            for k in ks:
                i, nt, w = scipy_iters(a.n, A, eps1, masks, k, nev, g, a.tol)
                its.append(i)
                tot.append(nt)
            out["scipy"][f"guard{g}"] = {"iters_first_nev": its, "iters_total": tot, "seconds": time.time() - t}
            print("scipy guard", g, its, tot, file=sys.stderr, flush=True)
    if "gpu" in a.which:
        from paper_2511_17107_b200 import api
        for v in a.variants.split(","):
            ctx = api.pc_create(A, a.n, eps1, masks)
            for key, val in VARIANTS[v].items():
                api.pc_set_option(ctx, key, val)
            r = api.pc_bands(ctx, ks, nev=nev, tol=a.tol, maxit=1000)
            out["gpu"][v] = {"iters": r["iters"].tolist(), "status": r["status"].tolist(),
                             "omega2_k0": r["omega2"][0][:4].tolist()}
            print("gpu", v, r["iters"].tolist(), file=sys.stderr, flush=True)
            ctx.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
