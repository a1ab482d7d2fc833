"""Regenerate the golden files under tests/golden/ from the CPU oracle ONLY.

Test infrastructure: imports ``oracle`` and ``synth`` and nothing from the CUDA path
(paper_2511_17107_b200/).  Every stored value is either a closed form typed from the paper
or the oracle's own eigensolve; the header of each file records the command and git hash.

  closed      c1_vacuum_n8.txt, homog_n8_R.txt  (closed forms, seconds)
  c2          SC sphere eps_lat = 13, n = 32, the full 33-point G-X-M-R-G path, 10 bands
  c3          SC-CURV pseudochiral, n = 64, 3 k-points of the path
  c4          FCC diamond pseudochiral, n = 128, X, L and one generic path point

Eigenvalues (c2-c4): O.eigs_iterative (SciPy LOBPCG on the oracle's sparse operator with the
oracle's own K_P^{-1}) to Res_j <= tol (absolute); the error of
an eigenvalue is <= Res^2 / gap (Rayleigh quotient of a residual-Res vector), ~1e-15 here.

usage: python tests/golden/gen_goldens.py {closed|c2|c3|c4} [--k i,j,..] [--jobs J] [--tol T]
  (each k-point runs in its own worker process; --jobs bounds the concurrency)
"""
from __future__ import annotations

import argparse
import math
import os
import subprocess
import sys
import time
from concurrent.futures import ProcessPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
GOLD = os.path.dirname(os.path.abspath(__file__))
PI = math.pi

# k-point indices on the synth.kpath paths (8 segments per edge)
SETS = {
    "c2": ("C2", None, 1e-8, 1000),                    # full path
    "c3": ("C3", [5, 8, 24], 1e-8, 600),               # generic G-X point, X(pi,0,0), R(pi,pi,pi)
    "c4": ("C4", [0, 13, 16], 2e-8, 400),              # X(0,2pi,0), generic U-L point, L(pi,pi,pi)
}


def _git():
    try:
        h = subprocess.run(["git", "-C", ROOT, "rev-parse", "--short=12", "HEAD"],
                           capture_output=True, text=True).stdout.strip()
        d = subprocess.run(["git", "-C", ROOT, "status", "--porcelain", "oracle", "synth"],
                           capture_output=True, text=True).stdout.strip()
        return h + ("+dirty(oracle/synth)" if d else "")
    except OSError:
        return "unknown"


def _solve(args):
    wname, ki, tol, maxiter = args
    import numpy as np
    import synth
    from oracle import pc_oracle as O
    w = synth.WORKLOADS[wname]
    k = w.kpoints()[ki]
    t = time.time()
    op = O.PenalizedOperator(w.n, k, w.A(), w.eps1(), w.masks(), "crossdof")
    info = {}
    ev, res = O.eigs_iterative(op, w.nev, tol=tol, seed=1000 + ki, maxiter=maxiter, guard=5, info=info)
    return ki, np.asarray(k), ev, res, info.get("iterations"), time.time() - t


def run_set(name, kidx, jobs, tol=None):
    import numpy as np
    import synth
    wname, default_k, dtol, maxiter = SETS[name]
    w = synth.WORKLOADS[wname]
    tol = dtol if tol is None else tol
    kidx = kidx or default_k or list(range(len(w.kpoints())))
    path = os.path.join(GOLD, f"{name}_{w.lattice}_{w.geometry}_n{w.n}.txt")
    done = {}
    with ProcessPoolExecutor(max_workers=jobs) as ex:
        for ki, k, ev, res, its, sec in ex.map(_solve, [(wname, i, tol, maxiter) for i in kidx]):
            done[ki] = (k, ev, res, its, sec)
            print(f"{name} k{ki} its={its} {sec:.0f}s maxres={res.max():.2e} ev={ev}", flush=True)
    # merge: rows of k-points not recomputed here are kept from an existing file (one file per set)
    old_rows, old_cmds = {}, []
    if os.path.exists(path):
        for line in open(path):
            if line.startswith("# Command:"):
                old_cmds.append(line.rstrip("\n"))
            elif line.strip() and not line.startswith("#"):
                key = line.split()[0]
                ki = int(key.lstrip("kevrsit")) if key[0] in "kers" or key.startswith("its") else None
                if ki is not None and ki not in done:
                    old_rows.setdefault(ki, []).append(line)
    with open(path, "w") as f:
        f.write(f"# {wname}: {w.lattice.upper()} {w.geometry}, eps1 '{w.eps}', n = {w.n}, {w.nev} smallest "
                f"eigenvalues of the penalised operator (PAPER.md:259, gamma rule P:457-462), CrossDoF.\n")
        f.write("# Source: oracle/pc_oracle.py eigs_iterative (SciPy LOBPCG on the oracle's sparse operator,\n"
                "#   oracle K_P^-1 preconditioner, guard 5, absolute Res_j tolerance as in each command, P:1059-1064).\n")
        for oc in old_cmds:
            f.write(oc + "\n")
        f.write(f"# Command: python tests/golden/gen_goldens.py {name} --k {','.join(map(str, kidx))} --tol {tol:g}"
                f"   git {_git()}   {time.strftime('%Y-%m-%d')}\n")
        f.write("# Rows: k<i> = k-point index on synth.kpath(lattice, 8) then kx ky kz; ev<i> = eigenvalues;\n"
                "#       res<i> = final oracle residual norms; its<i> = SciPy LOBPCG iterations.\n")
        for ki in sorted(old_rows):
            for line in old_rows[ki]:
                f.write(line)
        for ki in sorted(done):
            k, ev, res, its, _ = done[ki]
            f.write(f"k{ki} " + " ".join(f"{v:.17g}" for v in k) + "\n")
            f.write(f"ev{ki} " + " ".join(f"{v:.17g}" for v in ev) + "\n")
            f.write(f"res{ki} " + " ".join(f"{v:.3e}" for v in res) + "\n")
            f.write(f"its{ki} {its if its is not None else -1}\n")
    print("wrote", path)


def write_closed():
    """Closed forms: vacuum n=8 {|kappa|^2 x2, gamma|kappa|^2} (in the
    paper's D_0-averaged form mu = (4/h^2 + k^2) sin^2(pi m/N + atan(k h/2))) and the
    homogeneous pseudochiral medium per Fourier mode (App. A9 of SURVEY: with FULL masks M is a
    circulant whose per-mode 3x3 symbol is m_ii = eps_ii and t_ij = eps_ij * tau_ij(m), tau the
    symbol of T_ij; the per-mode operator is K_A M(m) K_A^H + gamma K_B)."""
    import numpy as np
    import synth

    def mu(n, k, m):
        h = 1.0 / n
        return (4 / h ** 2 + k ** 2) * np.sin(PI * m / n + np.arctan(k * h / 2)) ** 2

    n = 8
    rows = []
    for name, k in (("k_a", (PI, PI, PI)), ("k_b", (PI / 7, 3 * PI / 5, 4 * PI / 13))):
        m = np.arange(n)
        k2 = (mu(n, k[0], m)[None, None, :] + mu(n, k[1], m)[None, :, None] + mu(n, k[2], m)[:, None, None])
        k2 = k2.ravel()
        nk = math.sqrt(sum(c * c for c in k))
        gam = 4 * PI ** 2 if nk == 0 or nk >= 1 else 4 * PI ** 2 / nk ** 2
        vals = np.sort(np.concatenate([k2, k2, gam * k2]))[:6]
        rows.append(f"{name} " + " ".join(f"{v:.12f}" for v in vals))
    with open(os.path.join(GOLD, "c1_vacuum_n8.txt"), "w") as f:
        f.write("# SC vacuum, n=8, gamma = 4 pi^2, six smallest eigenvalues of the penalised operator.\n"
                "# Source: closed form {|kappa|^2 x2, gamma |kappa|^2} (PAPER.md:370-373) with the per-axis\n"
                "#   mu = (4/h^2 + k^2) sin^2(pi m/N + atan(k h/2)) of P:394.  k_a = (pi,pi,pi);\n"
                "#   k_b = (pi/7, 3pi/5, 4pi/13) (PAPER.md:1296).\n"
                f"# Command: python tests/golden/gen_goldens.py closed   git {_git()}\n")
        f.write("\n".join(rows) + "\n")

    # homogeneous medium: per mode, 3x3 symbol of the curl (K_A = [kappa]_x), of M (P:664-673 with
    # I_i = 1: M_ii = eps_ii, off-diagonal eps_ij (T_ij + T_ij)/2 = eps_ij T_ij), K_B = conj(k) k^T.
    # Symbols typed from P:182-193/P:241/P:274: lambda1(m) = (1 - e^{-2 pi i m/N})/h,
    # lambda0(m) = (1 + e^{-2 pi i m/N})/2; T12 = I (x) D0^T (x) D0 etc. (reading R5) has symbol
    # conj(lambda0(m_y)) lambda0(m_x).
    e1 = synth.eps_pseudochiral()
    out = []
    for lat in ("sc", "fcc"):
        A = synth.lattice(lat)
        B = np.linalg.inv(A)
        k = np.array([PI, PI, PI])
        th = 2 * PI * np.arange(n) / n
        l1 = (1 - np.exp(-1j * th)) * n
        l0 = (1 + np.exp(-1j * th)) / 2
        vals = []
        for m3 in range(n):
            for m2 in range(n):
                for m1 in range(n):
                    mm = (m1, m2, m3)
                    kap = np.array([sum(B[j, i] * l1[mm[j]] for j in range(3)) + 1j * k[i] * l0[mm[i]]
                                    for i in range(3)])
                    t12 = np.conj(l0[m2]) * l0[m1]
                    t13 = np.conj(l0[m3]) * l0[m1]
                    t23 = np.conj(l0[m3]) * l0[m2]
                    Mm = np.array([[e1[0, 0], e1[0, 1] * t12, e1[0, 2] * t13],
                                   [np.conj(e1[0, 1] * t12), e1[1, 1], e1[1, 2] * t23],
                                   [np.conj(e1[0, 2] * t13), np.conj(e1[1, 2] * t23), e1[2, 2]]])
                    KA = np.array([[0, -kap[2], kap[1]], [kap[2], 0, -kap[0]], [-kap[1], kap[0], 0]])
                    KB = np.conj(kap)[:, None] * kap[None, :]
                    vals.extend(np.linalg.eigvalsh(KA @ Mm @ KA.conj().T + 4 * PI ** 2 * KB))
        vals = np.sort(vals)[:10]
        out.append(f"{lat} " + " ".join(f"{v:.12f}" for v in vals))
    with open(os.path.join(GOLD, "homog_n8_R.txt"), "w") as f:
        f.write("# Homogeneous (FULL mask) pseudochiral medium, eps_1 = eps_pseudochiral(13, 0.875), CrossDoF,\n"
                "# n=8, k = (pi,pi,pi), gamma = 4 pi^2: ten smallest eigenvalues.\n"
                "# Source: per-mode closed form: eigenvalues of K_A(m) M(m) K_A(m)^H + gamma K_B(m) with the\n"
                "#   3x3 symbols typed from P:182-193, P:241 (reading R3), P:274, P:509-517, P:664-673 (reading R5).\n"
                f"# Command: python tests/golden/gen_goldens.py closed   git {_git()}\n")
        f.write("\n".join(out) + "\n")
    print("wrote closed-form goldens")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("which", choices=["closed", "c2", "c3", "c4"])
    ap.add_argument("--k", default="")
    ap.add_argument("--jobs", type=int, default=1)
    ap.add_argument("--tol", type=float, default=None)
    a = ap.parse_args()
    if a.which == "closed":
        write_closed()
        return
    kidx = [int(s) for s in a.k.split(",") if s.strip()]
    run_set(a.which, kidx, a.jobs, a.tol)


if __name__ == "__main__":
    main()
