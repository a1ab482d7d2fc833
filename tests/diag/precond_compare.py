"""Iteration counts of SciPy LOBPCG with the paper's K_P^{-1} vs the eps-weighted preconditioner
(DESIGN R16), oracle operator, C4 geometry at small n (test infrastructure: imports oracle/).
usage: python tests/diag/precond_compare.py [n]   (n = 16: 68/66/65 vs 37/34/34; n = 32: 72/74/80 vs 40/39/42)"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, scipy.sparse.linalg as spla
import synth
from oracle import pc_oracle as po
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
W = synth.WORKLOADS["C4"]
A = W.A(); masks = synth.make_masks(W.geometry, A, n); eps1 = W.eps1()
kp = synth.kpath(W.lattice, W.segments)
nev, guard, tol = 10, 6, 1e-5
for kk in [3, 17, 30]:
    k = kp[kk]
    op = po.PenalizedOperator(n, k, A, eps1, masks, "crossdof")
    kap = po.kappa_symbols(n, op.k, A).reshape(3, -1)  # (3, N^3)
    k2 = np.sum(np.abs(kap) ** 2, axis=0); k2s = np.where(k2 > 1e-28 * k2.max(), k2, 1.0)
    Md = op.M.diagonal().real
    def mv(X):
        X = np.asarray(X); return op.apply_fourier(X.T).T
    def kp_prec(X):
        X = np.asarray(X); return po.precond_fourier(n, op.k, A, op.gamma, X.T).T
    def kah(x):  # K_A^H x = -(conj kappa) x x ... = x x conj(kappa)
        x = x.reshape(3, -1); ck = np.conj(kap)
        return np.stack([x[1]*ck[2]-x[2]*ck[1], x[2]*ck[0]-x[0]*ck[2], x[0]*ck[1]-x[1]*ck[0]])
    def ka(s):  # K_A s = kappa x s
        return np.stack([kap[1]*s[2]-kap[2]*s[1], kap[2]*s[0]-kap[0]*s[2], kap[0]*s[1]-kap[1]*s[0]])
    def mpb_col(r):
        r3 = r.reshape(3, -1)
        u = kah(r) / k2s
        H = po.fft3_fourier_to_real(u.reshape(-1), n)
        H = H / Md
        s = po.fft3_real_to_fourier(H, n).reshape(3, -1)
        y = ka(s) / k2s
        kr = np.sum(kap * r3, axis=0)  # kappa^T r
        y = y + np.conj(kap) * kr / (op.gamma * k2s * k2s)
        y[:, k2 <= 1e-28 * k2.max()] = r3[:, k2 <= 1e-28 * k2.max()]
        return y.reshape(-1)
    def mpb_prec(X):
        X = np.asarray(X)
        return np.stack([mpb_col(X[:, j]) for j in range(X.shape[1])], axis=1)
    dim = op.dim
    Aop = spla.LinearOperator((dim, dim), matvec=lambda x: mv(x[:, None])[:, 0], matmat=mv, dtype=np.complex128)
    res = {}
    for name, pf in [("K_P", kp_prec), ("mpb", mpb_prec)]:
        Mop = spla.LinearOperator((dim, dim), matvec=lambda x, pf=pf: pf(x[:, None])[:, 0], matmat=pf, dtype=np.complex128)
        rng = np.random.default_rng(0)
        X0 = rng.standard_normal((dim, nev + guard)) + 1j * rng.standard_normal((dim, nev + guard))
        t = time.time()
        w, V, lh, rh = spla.lobpcg(Aop, X0, M=Mop, tol=tol, maxiter=400, largest=False, retLambdaHistory=True, retResidualNormsHistory=True)
        its = None
        for i, (lam, r) in enumerate(zip(lh, rh)):
            lam = np.asarray(lam); r = np.asarray(r)[:len(lam)]
            o = np.argsort(lam)[:nev]
            if np.all(r[o] <= tol): its = i; break
        res[name] = (its, len(lh), np.sort(w)[:3].round(6).tolist(), round(time.time()-t,1))
    print(n, kk, res, flush=True)
