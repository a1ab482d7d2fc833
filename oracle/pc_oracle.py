"""Plain, slow, obviously-correct CPU oracle (complex128, SciPy sparse) for

    Op = A_c M_eps A_c^H + gamma B^H B          (display:kc_formulation)

TEST INFRASTRUCTURE — only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg,
``--impl reference``) may import this module.  It shares no code with the CUDA path
(paper_2511_17107_b200/); its only common dependency is the input generator ``synth``.

Every function cites the PAPER.md passage it follows ("P:123" = PAPER.md line 123).  The
readings taken where the paper is silent, garbled or self-inconsistent are the ones listed in
DESIGN.md §Readings (= SURVEY.md §8(c)):

  R1  curl stencil sign typo P:163 -> matrix form P:203-204 is normative;
  R2  DFT convention: F_ij = w^{(i-1)(j-1)}/sqrt(N), w = exp(+2 pi i/N);
  R3  coordinate-transform blocks: Dhat_i = sum_j b_ji D_{1,j} + i k_i D_{0,i}  (P:241 read
      with the summation index on the derivative axis);
  R4  cross-DoF template P:647 duplicate term -> neighbours (i-1,j),(i-1,j+1),(i,j),(i,j+1);
  R5  Kronecker order of T_ij derived from the DoF geometry in the x-fastest
      layout of P:198: T12 = I (x) D0^T (x) D0, T13 = D0^T (x) I (x) D0, T23 = D0^T (x) D0 (x) I;
  R7  preconditioner modes with |kappa|^2 <= 1e-28 max|kappa|^2 pass through unchanged;
  R11 eigenvalues compared are those of the penalised operator;
  R12 at k = 0 (bitwise) the 3-dim null space is removed before taking nev.

Parity status of each function is recorded in DESIGN.md §Oracle pins; every function here is
pinned by a ``-m "not gpu"`` test in tests/test_oracle_pins.py (no "parity unpinned" items).
"""
from __future__ import annotations

import math

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

__all__ = [
    "circulant_D1", "circulant_D0", "circulant_symbols", "dft_matrix", "axis_embed",
    "shifted_blocks", "curl_matrix", "div_matrix", "transfer_T", "permittivity_matrix",
    "gamma_rule", "PenalizedOperator", "symbols_1d", "kappa_symbols", "precond_fourier",
    "precond_eps_fourier",
    "hpd_report", "eigs_dense", "eigs_iterative", "fft3_fourier_to_real",
    "fft3_real_to_fourier",
]


# ------------------------------------------------------------------------------------------
# 1-D circulants  (display:yee_circulantblock)
# ------------------------------------------------------------------------------------------

def circulant_D1(n: int) -> sp.csr_matrix:
    """D_1 = (1/h) [[1,..,-1],[-1,1,..],...]: (D_1 x)_r = (x_r - x_{r-1})/h, periodic."""
    h = 1.0 / n
    r = np.arange(n)
    rows = np.concatenate([r, r])
    cols = np.concatenate([r, (r - 1) % n])
    vals = np.concatenate([np.full(n, 1.0 / h), np.full(n, -1.0 / h)])
    return sp.csr_matrix((vals, (rows, cols)), shape=(n, n))


def circulant_D0(n: int) -> sp.csr_matrix:
    """D_0 = (1/2) [[1,..,1],[1,1,..],...]: (D_0 x)_r = (x_r + x_{r-1})/2, periodic."""
    r = np.arange(n)
    rows = np.concatenate([r, r])
    cols = np.concatenate([r, (r - 1) % n])
    return sp.csr_matrix((np.full(2 * n, 0.5), (rows, cols)), shape=(n, n))


def circulant_symbols(first_row: np.ndarray) -> np.ndarray:
    """Lemma 2.1: lambda_i = sum_j c_j w^{(i-1)(j-1)}, w = exp(2 pi i / N).
    Written as the explicit O(N^2) sum over the first row c."""
    c = np.asarray(first_row, dtype=np.complex128)
    n = c.size
    i = np.arange(n)[:, None]
    j = np.arange(n)[None, :]
    w = np.exp(2j * np.pi * (i * j % n) / n)
    return w @ c


def dft_matrix(n: int) -> np.ndarray:
    """F_ij = w^{(i-1)(j-1)} / sqrt(N), w = exp(2 pi i/N), unitary."""
    i = np.arange(n)[:, None]
    j = np.arange(n)[None, :]
    return np.exp(2j * np.pi * (i * j % n) / n) / math.sqrt(n)


# ------------------------------------------------------------------------------------------
# Kronecker embedding and shifted blocks
# ------------------------------------------------------------------------------------------

def axis_embed(D: sp.spmatrix, axis: int, n: int) -> sp.csr_matrix:
    """D_{s,1} = I_{N^2} (x) D_s, D_{s,2} = I_N (x) D_s (x) I_N, D_{s,3} = D_s (x) I_{N^2}.
    axis in {1,2,3}; axis 1 (x) is the last Kronecker factor = fastest index."""
    I = sp.identity(n, format="csr")
    if axis == 1:
        return sp.kron(sp.kron(I, I), D, format="csr")
    if axis == 2:
        return sp.kron(sp.kron(I, D), I, format="csr")
    if axis == 3:
        return sp.kron(sp.kron(D, I), I, format="csr")
    raise ValueError(axis)


def shifted_blocks(n: int, k, A) -> list:
    """Dhat_i = sum_j b_ji D_{1,j} + i k_i D_{0,i}, b = A^{-1} (reading R3).
    For A = I this is D_i = D_{1,i} + i k_i D_{0,i}."""
    k = np.asarray(k, dtype=np.float64)
    B = np.linalg.inv(np.asarray(A, dtype=np.float64))
    D1 = circulant_D1(n)
    D0 = circulant_D0(n)
    D1ax = [axis_embed(D1, j, n) for j in (1, 2, 3)]
    out = []
    for i in range(3):
        M = sum(B[j, i] * D1ax[j] for j in range(3)).astype(np.complex128)
        M = M + 1j * k[i] * axis_embed(D0, i + 1, n)
        out.append(M.tocsr())
    return out


def curl_matrix(n: int, k, A) -> sp.csr_matrix:
    """Outer curl A_c : E_h -> F_h (display:yee_ABmatrix, with blocks Dhat_i):
        [[0, -D3, D2], [D3, 0, -D1], [-D2, D1, 0]]."""
    D1, D2, D3 = shifted_blocks(n, k, A)
    return sp.bmat([[None, -D3, D2], [D3, None, -D1], [-D2, D1, None]], format="csr")


def div_matrix(n: int, k, A) -> sp.csr_matrix:
    """Shifted divergence B : F_h -> V_h, B = [D1 D2 D3]."""
    D1, D2, D3 = shifted_blocks(n, k, A)
    return sp.hstack([D1, D2, D3], format="csr")


# ------------------------------------------------------------------------------------------
# Permittivity
# ------------------------------------------------------------------------------------------

def transfer_T(n: int) -> tuple:
    """Cross-DoF transfer matrices under readings R4/R5:
    T12 = I (x) D0^T (x) D0, T13 = D0^T (x) I (x) D0, T23 = D0^T (x) D0 (x) I."""
    D0 = circulant_D0(n)
    I = sp.identity(n, format="csr")
    T12 = sp.kron(sp.kron(I, D0.T), D0, format="csr")
    T13 = sp.kron(sp.kron(D0.T, I), D0, format="csr")
    T23 = sp.kron(sp.kron(D0.T, D0), I, format="csr")
    return T12, T13, T23


def permittivity_matrix(eps1, masks, mode: str = "crossdof") -> sp.csr_matrix:
    """Discrete inverse-permittivity matrix M_eps (3N^3 x 3N^3).

    Diagonal blocks M_ii = (eps_ii - 1) I_i + I.
    mode "diagonal": off-diagonal blocks zero (requires eps offdiag = 0).
    mode "trivial":  off-diagonal blocks eps_ij I_V.
    mode "crossdof": off-diagonal blocks eps_ij S_ij, S_ij = (I_i T_ij + T_ij I_j)/2.
    masks: uint8 (4, n, n, n) = (I1, I2, I3, IV) each [z][y][x].
    """
    eps1 = np.asarray(eps1, dtype=np.complex128)
    masks = np.asarray(masks)
    n = masks.shape[-1]
    Ii = [sp.diags(masks[c].reshape(-1).astype(np.float64)) for c in range(3)]
    IV = sp.diags(masks[3].reshape(-1).astype(np.float64))
    Id = sp.identity(n ** 3, format="csr")
    blocks = [[None] * 3 for _ in range(3)]
    for i in range(3):
        blocks[i][i] = ((eps1[i, i].real - 1.0) * Ii[i] + Id).astype(np.complex128)
    if mode == "diagonal":
        if np.any(np.abs(eps1 - np.diag(np.diag(eps1))) != 0):
            raise ValueError("diagonal mode requires a diagonal eps1")
    elif mode == "trivial":
        for i in range(3):
            for j in range(i + 1, 3):
                blocks[i][j] = eps1[i, j] * IV
                blocks[j][i] = np.conj(eps1[i, j]) * IV
    elif mode == "crossdof":
        T = {(0, 1): None, (0, 2): None, (1, 2): None}
        T[(0, 1)], T[(0, 2)], T[(1, 2)] = transfer_T(n)
        for (i, j), Tij in T.items():
            S = 0.5 * (Ii[i] @ Tij + Tij @ Ii[j])
            blocks[i][j] = eps1[i, j] * S
            blocks[j][i] = np.conj(eps1[i, j]) * S.T
    else:
        raise ValueError(mode)
    return sp.bmat(blocks, format="csr").astype(np.complex128)


def hpd_report(eps1) -> dict:
    """Assumptions 1-3 and the guarantees they give (Props)."""
    e = np.asarray(eps1, dtype=np.complex128)
    ev = np.linalg.eigvalsh(e)
    a1 = bool(ev.min() > 0 and ev.max() <= 1.0 + 1e-15)
    a2 = bool(all(e[i, i].real > sum(abs(e[i, j]) for j in range(3) if j != i) for i in range(3)))
    a3 = bool(any(e[i, j] == 0 for i in range(3) for j in range(3) if i != j))
    return {"assumption1": a1, "sdd": a2, "zero_offdiag": a3, "guaranteed": a1 and (a2 or a3)}


# ------------------------------------------------------------------------------------------
# Penalty and the assembled operator
# ------------------------------------------------------------------------------------------

def gamma_rule(k) -> float:
    """Practical penalty: 4 pi^2 if k = 0 or ||k|| > 1, 4 pi^2 / ||k||^2 if
    ||k|| in (0,1).  (||k|| = 1 exactly: both branches give 4 pi^2.)"""
    k = np.asarray(k, dtype=np.float64)
    nk = float(np.linalg.norm(k))
    if nk == 0.0 or nk >= 1.0:
        return 4.0 * math.pi ** 2
    return 4.0 * math.pi ** 2 / nk ** 2


class PenalizedOperator:
    """Op = A_c M A_c^H + gamma B^H B kept as a product of sparse factors."""

    def __init__(self, n, k, A, eps1, masks, mode="crossdof", gamma=None):
        self.n = int(n)
        self.k = np.asarray(k, dtype=np.float64)
        self.A = np.asarray(A, dtype=np.float64)
        self.gamma = gamma_rule(self.k) if gamma is None else float(gamma)
        self.Ac = curl_matrix(self.n, self.k, self.A)
        self.AcH = self.Ac.conj().T.tocsr()
        self.B = div_matrix(self.n, self.k, self.A)
        self.BH = self.B.conj().T.tocsr()
        self.M = permittivity_matrix(eps1, masks, mode)

    @property
    def dim(self) -> int:
        return 3 * self.n ** 3

    def apply_real(self, H: np.ndarray) -> np.ndarray:
        """y = Op H for real-space face fields H (3N^3,) or (3N^3, m)."""
        return self.Ac @ (self.M @ (self.AcH @ H)) + self.gamma * (self.BH @ (self.B @ H))

    def matrix(self) -> sp.csr_matrix:
        return (self.Ac @ self.M @ self.AcH + self.gamma * (self.BH @ self.B)).tocsr()

    def dense(self) -> np.ndarray:
        return self.matrix().toarray()

    def apply_fourier(self, xhat: np.ndarray) -> np.ndarray:
        """y_hat = F3^H Op F3 x_hat with x_hat = F3^H H.  Input/output blocks are
        (ncols, 3N^3) (column-major block, ld = 3N^3)."""
        X = np.atleast_2d(xhat)
        out = np.empty_like(X, dtype=np.complex128)
        for c in range(X.shape[0]):
            H = fft3_fourier_to_real(X[c], self.n)
            out[c] = fft3_real_to_fourier(self.apply_real(H), self.n)
        return out.reshape(np.shape(xhat))


def fft3_fourier_to_real(x: np.ndarray, n: int) -> np.ndarray:
    """H = F3 x: F (w = e^{+2 pi i/N}, unitary) on all three axes of each component,
    = numpy ifftn(norm="ortho")."""
    v = np.asarray(x, dtype=np.complex128).reshape(3, n, n, n)
    return np.fft.ifftn(v, axes=(1, 2, 3), norm="ortho").reshape(-1)


def fft3_real_to_fourier(H: np.ndarray, n: int) -> np.ndarray:
    """x = F3^H H = numpy fftn(norm="ortho") per component."""
    v = np.asarray(H, dtype=np.complex128).reshape(3, n, n, n)
    return np.fft.fftn(v, axes=(1, 2, 3), norm="ortho").reshape(-1)


# ------------------------------------------------------------------------------------------
# Fourier symbols and the preconditioner
# ------------------------------------------------------------------------------------------

def symbols_1d(n: int):
    """Diagonals Lambda_1, Lambda_0 of D_1 = F Lambda_1 F^H, D_0 = F Lambda_0 F^H from Lemma 2.1
    applied to their first rows."""
    h = 1.0 / n
    r1 = np.zeros(n)
    r1[0], r1[-1] = 1.0 / h, -1.0 / h
    r0 = np.zeros(n)
    r0[0], r0[-1] = 0.5, 0.5
    return circulant_symbols(r1), circulant_symbols(r0)


def kappa_symbols(n: int, k, A) -> np.ndarray:
    """Per-mode symbols kappa_i(m) of Dhat_i (P:495-503 with reading R3), shape (3, n, n, n)
    indexed [i][m3][m2][m1]."""
    k = np.asarray(k, dtype=np.float64)
    B = np.linalg.inv(np.asarray(A, dtype=np.float64))
    l1, l0 = symbols_1d(n)
    # axis j symbol broadcast into [m3][m2][m1]
    def on_axis(t, j):
        shape = [1, 1, 1]
        shape[2 - j] = n
        return t.reshape(shape)
    kap = np.zeros((3, n, n, n), dtype=np.complex128)
    for i in range(3):
        for j in range(3):
            kap[i] = kap[i] + B[j, i] * on_axis(l1, j)
        kap[i] = kap[i] + 1j * k[i] * on_axis(l0, i)
    return kap


def precond_fourier(n: int, k, A, gamma: float, R: np.ndarray) -> np.ndarray:
    """P = K_P^{-1} R per Fourier mode, K_P = K_A K_A^H + gamma K_B with
    K_A = [kappa]_x and K_B = conj(kappa) kappa^T, assembled as explicit
    3x3 matrices and solved mode by mode.  Modes with |kappa|^2 <= 1e-28 max pass through
    (reading R7).  R: (ncols, 3N^3)."""
    kap = kappa_symbols(n, k, A).reshape(3, -1).T  # (N^3, 3)
    nm = kap.shape[0]
    KA = np.zeros((nm, 3, 3), dtype=np.complex128)
    KA[:, 0, 1], KA[:, 0, 2] = -kap[:, 2], kap[:, 1]
    KA[:, 1, 0], KA[:, 1, 2] = kap[:, 2], -kap[:, 0]
    KA[:, 2, 0], KA[:, 2, 1] = -kap[:, 1], kap[:, 0]
    KB = np.conj(kap)[:, :, None] * kap[:, None, :]
    KP = KA @ np.conj(np.transpose(KA, (0, 2, 1))) + gamma * KB
    k2 = np.sum(np.abs(kap) ** 2, axis=1)
    zero = k2 <= 1e-28 * k2.max()
    KP[zero] = np.eye(3)
    Rb = np.atleast_2d(R)
    out = np.empty_like(Rb, dtype=np.complex128)
    for c in range(Rb.shape[0]):
        v = Rb[c].reshape(3, -1).T[:, :, None]
        out[c] = np.linalg.solve(KP, v)[:, :, 0].T.reshape(-1)
    return out.reshape(np.shape(R))


def precond_eps_fourier(n: int, k, A, gamma: float, eps1, masks, mode: str, R: np.ndarray) -> np.ndarray:
    """eps-weighted preconditioner (BEYOND THE PAPER: the paper's preconditioner is K_P^{-1},
    P:530-548; this is the Maxwell-solver variant that weights the two curl halves by the medium,
    reading R16 in DESIGN.md).  Per column r (Fourier coordinates):

        T r = K_A^{+H} F3^H D^{-1} F3 K_A^{+} r + Pi r / (gamma |kappa|^2)

    with K_A = [kappa]_x, its pseudo-inverse K_A^+ = K_A^H / |kappa|^2, the projector
    Pi = conj(kappa) kappa^T / |kappa|^2 onto the range of K_B, F3 = ifftn and
    D = the diagonal of the oracle's own M_eps (permittivity_matrix).  Modes with
    |kappa|^2 <= 1e-28 max|kappa|^2 map to 0.  R: (ncols, 3N^3)."""
    kap = kappa_symbols(n, k, A).reshape(3, -1)           # (3, N^3)
    k2 = np.sum(np.abs(kap) ** 2, axis=0)
    zero = k2 <= 1e-28 * k2.max()
    k2s = np.where(zero, 1.0, k2)
    nm = kap.shape[1]
    # explicit 3x3 matrices per mode
    KA = np.zeros((nm, 3, 3), dtype=np.complex128)
    KA[:, 0, 1], KA[:, 0, 2] = -kap[2], kap[1]
    KA[:, 1, 0], KA[:, 1, 2] = kap[2], -kap[0]
    KA[:, 2, 0], KA[:, 2, 1] = -kap[1], kap[0]
    KAp = np.conj(np.transpose(KA, (0, 2, 1))) / k2s[:, None, None]      # K_A^+
    KApH = np.conj(np.transpose(KAp, (0, 2, 1)))                          # K_A^{+H}
    Pi = np.conj(kap).T[:, :, None] * kap.T[:, None, :] / k2s[:, None, None]
    Dinv = 1.0 / permittivity_matrix(eps1, masks, mode).diagonal()
    Rb = np.atleast_2d(R)
    out = np.empty_like(Rb, dtype=np.complex128)
    for c in range(Rb.shape[0]):
        r = Rb[c].reshape(3, -1).T[:, :, None]                            # (N^3, 3, 1)
        u = (KAp @ r)[:, :, 0].T.reshape(-1)                              # K_A^+ r
        H = fft3_fourier_to_real(u, n) * Dinv                             # D^{-1} F3 (.)
        s = fft3_real_to_fourier(H, n).reshape(3, -1).T[:, :, None]       # F3^H (.)
        y = (KApH @ s)[:, :, 0] + (Pi @ r)[:, :, 0] / (gamma * k2s[:, None])
        y[zero] = 0.0
        out[c] = y.T.reshape(-1)
    return out.reshape(np.shape(R))


# ------------------------------------------------------------------------------------------
# Eigenvalues
# ------------------------------------------------------------------------------------------

def _is_gamma_point(k) -> bool:
    return bool(np.all(np.asarray(k, dtype=np.float64) == 0.0))


def eigs_dense(op: PenalizedOperator, nev: int) -> np.ndarray:
    """The nev smallest eigenvalues of the dense penalised operator.  At k = 0 the
    3 null-space eigenvalues are removed first (reading R12)."""
    w = np.linalg.eigvalsh(op.dense())
    if _is_gamma_point(op.k):
        w = w[3:]
    return w[:nev]


def eigs_iterative(op: PenalizedOperator, nev: int, tol: float = 1e-8, seed: int = 0,
                   maxiter: int = 2000, guard: int = 5, info: dict | None = None):
    """The nev smallest eigenvalues of the penalised operator by SciPy's LOBPCG (library
    primitive) in Fourier coordinates with the oracle's own K_P^{-1} as
    preconditioner.  At k = 0 the null space (constant fields; in Fourier
    coordinates the three zero-mode unit vectors) is passed as a constraint (reading R12).
    Returns (eigenvalues, residual norms ||Op x - w x|| per P:1059-1062).  If ``info`` is a
    dict, the number of LOBPCG iterations SciPy ran is stored in info["iterations"]."""
    n = op.n
    dim = op.dim
    gamma = op.gamma

    def mv(X):
        X = np.asarray(X)
        if X.ndim == 1:
            return op.apply_fourier(X[None, :])[0]
        return op.apply_fourier(X.T).T

    def pc(X):
        X = np.asarray(X)
        if X.ndim == 1:
            return precond_fourier(n, op.k, op.A, gamma, X[None, :])[0]
        return precond_fourier(n, op.k, op.A, gamma, X.T).T

    Aop = spla.LinearOperator((dim, dim), matvec=mv, matmat=mv, dtype=np.complex128)
    Mop = spla.LinearOperator((dim, dim), matvec=pc, matmat=pc, dtype=np.complex128)
    rng = np.random.default_rng(seed)
    m = nev + guard
    X0 = rng.standard_normal((dim, m)) + 1j * rng.standard_normal((dim, m))
    Y = None
    if _is_gamma_point(op.k):
        Y = np.zeros((dim, 3), dtype=np.complex128)
        for c in range(3):
            Y[c * n ** 3, c] = 1.0
        X0[[0, n ** 3, 2 * n ** 3], :] = 0.0
    if info is None:
        w, V = spla.lobpcg(Aop, X0, M=Mop, Y=Y, tol=tol, maxiter=maxiter, largest=False)
    else:
        w, V, hist = spla.lobpcg(Aop, X0, M=Mop, Y=Y, tol=tol, maxiter=maxiter, largest=False,
                                 retResidualNormsHistory=True)
        info["iterations"] = len(hist)
    order = np.argsort(w)
    w, V = w[order], V[:, order]
    R = mv(V) - V * w[None, :]
    res = np.linalg.norm(R, axis=0) / np.linalg.norm(V, axis=0)
    return w[:nev], res[:nev]
