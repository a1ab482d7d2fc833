"""Library-composition baseline of the Fourier-space apply (SURVEY §8(d) "comparison baselines"): the
paper's own GPU recipe -- batched 3-D FFTs from the vendor library (cuFFT through torch.fft) plus
separate elementwise kernels for the symbol products and the CrossDoF stencil (P:523-529,
P:545-548) -- on the same B200, so the fused pc_apply can be compared against it.

This is a comparison arm only: nothing in the library path imports it.  It materialises the
symbol arrays kappa_i(m) (3 N^3 complex) and uses torch.roll for the 4-point averages T_ij.

  u = x^ x conj(kappa);  v = ifftn(u, ortho);  w = M_eps v;  s = fftn(w, ortho)
  y = kappa x s + gamma conj(kappa) (kappa . x^)
"""
import math

import numpy as np
import torch


def _symbols(n):
    m = np.arange(n)
    w = np.exp(-2j * math.pi * m / n)
    return (1.0 - w) * n, 0.5 * (1.0 + w)  # lambda_1 (h = 1/n), lambda_0


def kappa(n, k, A, device):
    """kappa_i(m) = sum_j b_ji lambda_1(m_j) + i k_i lambda_0(m_i), arrays [m3][m2][m1]."""
    B = np.linalg.inv(np.asarray(A, dtype=np.float64).reshape(3, 3))
    l1, l0 = _symbols(n)
    axes = [l1.reshape(1, 1, n), l1.reshape(1, n, 1), l1.reshape(n, 1, 1)]
    axes0 = [l0.reshape(1, 1, n), l0.reshape(1, n, 1), l0.reshape(n, 1, 1)]
    out = []
    for i in range(3):
        v = np.zeros((n, n, n), dtype=np.complex128)
        for j in range(3):
            v = v + B[j, i] * axes[j]
        v = v + 1j * k[i] * axes0[i]
        out.append(torch.from_numpy(v).to(device))
    return out


def _avg(E, sx, sy, sz):
    """1/4 sum over two shifts on two axes: each (axis, s) pair averages E and E rolled by s."""
    for dim, s in ((-1, sx), (-2, sy), (-3, sz)):
        if s:
            E = E + torch.roll(E, shifts=s, dims=dim)
    return 0.25 * E


class LibraryApply:
    def __init__(self, n, A, k, eps1, masks, gamma, device):
        self.n = n
        self.k3 = kappa(n, np.asarray(k, dtype=np.float64), A, device)
        self.kc = [t.conj() for t in self.k3]
        mk = torch.from_numpy(np.asarray(masks, dtype=np.float64)).to(device)
        self.I = [mk[c] for c in range(3)]
        e = np.asarray(eps1, dtype=np.complex128)
        self.e = e
        self.m = [(e[c, c].real - 1.0) * self.I[c] + 1.0 for c in range(3)]
        self.gamma = float(gamma)

    # T_ij E and T_ij^T E (x-fastest Kronecker forms I(x)D0^T(x)D0 etc.; D0 averages r-1, r)
    # roll(+1) brings index r-1 to r; roll(-1) brings r+1.
    def T(self, ij, E, transpose=False):
        s = -1 if transpose else 1
        if ij == (0, 1):
            return _avg(E, s, -s, 0)   # x: (i-1, i), y: (j, j+1)
        if ij == (0, 2):
            return _avg(E, s, 0, -s)   # x: (i-1, i), z: (k, k+1)
        return _avg(E, 0, s, -s)       # (1, 2): y: (j-1, j), z: (k, k+1)

    def eps(self, v):
        e, I = self.e, self.I
        w = [self.m[c] * v[c] for c in range(3)]
        for (i, j) in ((0, 1), (0, 2), (1, 2)):
            if e[i, j] == 0:
                continue
            Sv = 0.5 * (I[i] * self.T((i, j), v[j]) + self.T((i, j), I[j] * v[j]))
            STv = 0.5 * (self.T((i, j), I[i] * v[i], True) + I[j] * self.T((i, j), v[i], True))
            w[i] = w[i] + complex(e[i, j]) * Sv
            w[j] = w[j] + complex(np.conj(e[i, j])) * STv
        return w

    def __call__(self, X):
        n = self.n
        x = X.view(X.shape[0], 3, n, n, n)
        x1, x2, x3 = x[:, 0], x[:, 1], x[:, 2]
        c1, c2, c3 = self.kc
        u = torch.stack([x2 * c3 - x3 * c2, x3 * c1 - x1 * c3, x1 * c2 - x2 * c1], dim=1)
        v = torch.fft.ifftn(u, dim=(-3, -2, -1), norm="ortho")
        w = self.eps([v[:, 0], v[:, 1], v[:, 2]])
        s = torch.fft.fftn(torch.stack(w, dim=1), dim=(-3, -2, -1), norm="ortho")
        k1, k2, k3 = self.k3
        s1, s2, s3 = s[:, 0], s[:, 1], s[:, 2]
        kx = k1 * x1 + k2 * x2 + k3 * x3
        g = self.gamma
        y = torch.stack([k2 * s3 - k3 * s2 + g * c1 * kx,
                         k3 * s1 - k1 * s3 + g * c2 * kx,
                         k1 * s2 - k2 * s1 + g * c3 * kx], dim=1)
        return y.reshape(X.shape[0], 3 * n ** 3)
