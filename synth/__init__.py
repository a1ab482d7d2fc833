"""Seeded synthetic inputs shared by the CUDA path's tests/bench and by the CPU oracle.

This module holds NONE of the method's arithmetic (no difference operators, symbols,
permittivity discretisation, penalty rule or eigensolver).  It only produces the
*inputs* of the problem stated in PAPER.md:

* lattice vectors a_1..a_3                        (display:exp_latticeconst)
* Brillouin-zone symmetry points and k-paths      (display:exp_bzsym)
* the inverse-permittivity tensor eps_1           (display:exp_permittivity;
                                                   PAPER.md:1285 for the ill-conditioned case)
* rasterised indicator masks I_1, I_2, I_3, I_V   (display:permittivity_indicatormatrix;
                                                   geometries PAPER.md:1034-1053)
* seeded complex test vectors.

Readings of the paper used here are listed in DESIGN.md ("Readings") and SURVEY.md §8(c):
FCC U point fixed to (pi/2, 2pi, pi/2) (reading 9), SC-CURV cylinders along the body diagonals
(reading 8), FCC diamond spheroids with semi-minor axis 0.11 (reading 8), DoF sample points
(reading 6).

Layout conventions: a scalar grid function is an array [z][y][x] (x fastest),
a field is [c][z][y][x]; a block of ncols fields is C-contiguous (ncols, 3*N^3), i.e. column-major
with leading dimension 3*N^3.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

PI = math.pi

# --------------------------------------------------------------------------------------
# Lattices
# --------------------------------------------------------------------------------------


def lattice(kind: str) -> np.ndarray:
    """Return A = (a_1, a_2, a_3) as a 3x3 array whose COLUMNS are the primitive vectors.

    PAPER.md:965-971 (display:exp_latticeconst).  Row-major flattening of this matrix is the
    ``A[9]`` argument of ``pc_create``.
    """
    kind = kind.lower()
    if kind == "sc":
        cols = [(1, 0, 0), (0, 1, 0), (0, 0, 1)]
    elif kind == "fcc":
        cols = [(0, 0.5, 0.5), (0.5, 0, 0.5), (0.5, 0.5, 0)]
    elif kind == "bcc":
        cols = [(-0.5, 0.5, 0.5), (0.5, -0.5, 0.5), (0.5, 0.5, -0.5)]
    else:
        raise ValueError(f"unknown lattice {kind!r}")
    return np.array(cols, dtype=np.float64).T.copy()


# --------------------------------------------------------------------------------------
# Symmetry points and k-paths
# --------------------------------------------------------------------------------------


def symmetry_points(kind: str) -> dict:
    """Labelled Brillouin-zone points, Cartesian, lattice constant 1.

    SC labels: the paper's L(pi,0,0), M(pi,pi,0), N(pi,pi,pi) are the
    standard X, M, R; both names are provided.  FCC U is read as (pi/2, 2pi, pi/2)
    (PAPER.md:983 prints (pi/2, 2pi, pi), outside the first BZ).
    """
    kind = kind.lower()
    if kind == "sc":
        p = {"G": (0, 0, 0), "X": (PI, 0, 0), "M": (PI, PI, 0), "R": (PI, PI, PI)}
        p.update({"L": p["X"], "N": p["R"]})
    elif kind == "fcc":
        p = {"X": (0, 2 * PI, 0), "U": (PI / 2, 2 * PI, PI / 2), "L": (PI, PI, PI),
             "G": (0, 0, 0), "W": (PI, 2 * PI, 0), "K": (1.5 * PI, 1.5 * PI, 0)}
    elif kind == "bcc":
        p = {"H'": (2 * PI, 0, 0), "G": (0, 0, 0), "P": (PI, PI, PI), "N": (PI, 0, PI),
             "H": (0, 2 * PI, 0)}
    else:
        raise ValueError(kind)
    return {k: np.array(v, dtype=np.float64) for k, v in p.items()}


DEFAULT_PATHS = {
    "sc": ["G", "X", "M", "R", "G"],
    "fcc": ["X", "U", "L", "G", "X", "W", "K"],
    "bcc": ["H'", "G", "P", "N", "H"],
}


def kpath(kind: str, segments: int, labels=None) -> np.ndarray:
    """Uniform linear interpolation between consecutive symmetry points (SPEC build_kpath);
    anchors appear once; count = n_anchor + (n_anchor-1)*(segments-1).  Returns (nk, 3)."""
    pts = symmetry_points(kind)
    labels = labels or DEFAULT_PATHS[kind.lower()]
    if len(labels) < 2 or segments < 1:
        raise ValueError("need >=2 anchors and segments>=1")
    out = [pts[labels[0]]]
    for a, b in zip(labels[:-1], labels[1:]):
        pa, pb = pts[a], pts[b]
        for s in range(1, segments + 1):
            out.append(pa + (pb - pa) * (s / segments))
    return np.array(out, dtype=np.float64)


# --------------------------------------------------------------------------------------
# Inverse-permittivity tensors
# --------------------------------------------------------------------------------------


def eps_isotropic(eps_lattice: float = 13.0) -> np.ndarray:
    """eps_1 = eps_lattice^{-1} I_3."""
    return np.eye(3, dtype=np.complex128) / eps_lattice


def eps_pseudochiral(eps_lattice: float = 13.0, beta: float = 0.875) -> np.ndarray:
    """eps_1 = eps_lattice^{-1} [[sqrt(1+b^2), -i b, 0], [i b, sqrt(1+b^2), 0], [0, 0, 1]]
    (beta = 0.875 PAPER.md:1090)."""
    b = abs(beta)
    s = math.sqrt(1.0 + b * b)
    e = np.array([[s, -1j * b, 0], [1j * b, s, 0], [0, 0, 1]], dtype=np.complex128)
    return e / eps_lattice


def eps_sdd() -> np.ndarray:
    """A strictly-diagonally-dominant Hermitian eps_1 with all off-diagonals non-zero
    (satisfies Assumptions 1+2; SURVEY §8(d) stencil-generality input)."""
    return np.array([[0.5, 0.1 + 0.05j, 0.05 - 0.1j],
                     [0.1 - 0.05j, 0.4, 0.08j],
                     [0.05 + 0.1j, -0.08j, 0.3]], dtype=np.complex128)


def eps_extreme(seed: int = 7) -> np.ndarray:
    """eps_1 = U diag(1e-1, 1e-3, 1e-5) U^H with U a seeded random unitary."""
    rng = np.random.default_rng(seed)
    z = rng.standard_normal((3, 3)) + 1j * rng.standard_normal((3, 3))
    q, r = np.linalg.qr(z)
    q = q * (np.diag(r) / np.abs(np.diag(r)))
    e = q @ np.diag([1e-1, 1e-3, 1e-5]) @ q.conj().T
    return 0.5 * (e + e.conj().T)


# --------------------------------------------------------------------------------------
# Geometry rasterisation  (PAPER.md:596-605 indicators; PAPER.md:1034-1053 shapes)
# --------------------------------------------------------------------------------------

# Sample points of the four DoF families, as fractional offsets (in units of h) added to the
# 0-based array index (a, b, c) = (x, y, z).  1-based labels (i, j, k) = (a+1, b+1, c+1);
# E^1_{i-1/2,j,k} sits at ((i-1/2)h, jh, kh).
DOF_OFFSETS = {
    "I1": (0.5, 1.0, 1.0),
    "I2": (1.0, 0.5, 1.0),
    "I3": (1.0, 1.0, 0.5),
    "IV": (0.5, 0.5, 0.5),
}


def _frac_points(n: int, off) -> np.ndarray:
    h = 1.0 / n
    c, b, a = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    x = (a + off[0]) * h
    y = (b + off[1]) * h
    z = (c + off[2]) * h
    return np.stack([x, y, z], axis=-1)  # [z][y][x][3]


def _min_image(v: np.ndarray) -> np.ndarray:
    """Minimum-image displacement for the cubic period-1 structure (conventional cell)."""
    return v - np.round(v)


def _in_sphere(p, c, r):
    v = _min_image(p - c)
    return np.sum(v * v, axis=-1) <= r * r


def _in_cylinder(p, c, d, r):
    """Infinite cylinder of radius r along direction d through c; all 27 nearest line images
    are tested (the minimum image of a point is not the nearest image of a line)."""
    d = d / np.linalg.norm(d)
    hit = np.zeros(p.shape[:-1], dtype=bool)
    v0 = _min_image(p - c)
    for n in np.ndindex(3, 3, 3):
        v = v0 - (np.array(n, dtype=np.float64) - 1.0)
        t = v @ d
        hit |= (np.sum(v * v, axis=-1) - t * t) <= r * r
    return hit


def _in_spheroid(p, f1, f2, b):
    """Prolate spheroid with foci f1, f2 and semi-minor axis b: |p-f1|+|p-f2| <= 2a,
    a^2 = b^2 + c^2, c = |f1-f2|/2 (minimum image about the centre; extent < 1/2)."""
    half = 0.5 * (f2 - f1)
    c = np.linalg.norm(half)
    a = math.sqrt(b * b + c * c)
    v = _min_image(p - 0.5 * (f1 + f2))
    d1 = np.sqrt(np.sum((v + half) ** 2, axis=-1))
    d2 = np.sqrt(np.sum((v - half) ** 2, axis=-1))
    return d1 + d2 <= 2 * a


def _diamond_objects():
    """Diamond structure in the conventional cubic cell (side 1): FCC sites x basis
    {(0,0,0), (1/4,1/4,1/4)} (reading SURVEY §8(c) item 8)."""
    fcc = [np.array(s, dtype=np.float64) for s in
           [(0, 0, 0), (0, 0.5, 0.5), (0.5, 0, 0.5), (0.5, 0.5, 0)]]
    bonds_dir = [np.array(v) * 0.25 for v in [(1, 1, 1), (-1, -1, 1), (-1, 1, -1), (1, -1, -1)]]
    atoms, bonds = [], []
    for s in fcc:
        atoms.append(s)
        atoms.append(s + 0.25)
        for v in bonds_dir:
            bonds.append((s, s + v))
    return atoms, bonds


def contains(kind: str, p: np.ndarray, A: np.ndarray, params: dict | None = None) -> np.ndarray:
    """Membership of Cartesian points p[..., 3] in Omega_1 (with periodic images)."""
    params = params or {}
    kind = kind.lower()
    shape = p.shape[:-1]
    if kind == "vacuum":
        return np.zeros(shape, dtype=bool)
    if kind == "full":
        return np.ones(shape, dtype=bool)
    if kind in ("bcc_sg", "bcc_dg"):
        t = params.get("threshold", 1.1)
        x, y, z = (2 * PI * p[..., 0], 2 * PI * p[..., 1], 2 * PI * p[..., 2])
        g = np.sin(x) * np.cos(y) + np.sin(y) * np.cos(z) + np.sin(z) * np.cos(x)
        return g > t if kind == "bcc_sg" else np.abs(g) > t
    inside = np.zeros(shape, dtype=bool)
    if kind == "sphere":
        r = params.get("radius", 0.345)
        return _in_sphere(p, np.full(3, 0.5), r)
    if kind == "sc_curv":
        r = params.get("radius", 0.345)
        rc = params.get("cyl_radius", 0.11)
        ctr = np.full(3, 0.5)
        dirs = [np.array(v, dtype=np.float64) for v in [(1, 1, 1), (-1, 1, 1), (1, -1, 1), (1, 1, -1)]]
        inside |= _in_sphere(p, ctr, r)
        for d in dirs:
            inside |= _in_cylinder(p, ctr, d, rc)
        return inside
    if kind == "fcc_diamond":
        r = params.get("radius", 0.12)
        b = params.get("minor", 0.11)
        atoms, bonds = _diamond_objects()
        for a in atoms:
            inside |= _in_sphere(p, a, r)
        for f1, f2 in bonds:
            inside |= _in_spheroid(p, f1, f2, b)
        return inside
    raise ValueError(f"unknown geometry {kind!r}")


def make_masks(kind: str, A: np.ndarray, n: int, params: dict | None = None,
               seed: int | None = None) -> np.ndarray:
    """Rasterise a geometry into uint8 indicator masks, shape (4, n, n, n) = (I1, I2, I3, IV),
    each [z][y][x].  Pointwise evaluation at the DoF location, fractional
    coordinates mapped to Cartesian p = A x (SPEC geometry design decision).

    kind "random" draws seeded Bernoulli(0.5) masks (test input with every stencil pattern).
    """
    if kind == "random":
        rng = np.random.default_rng(seed if seed is not None else 0)
        fill = (params or {}).get("fill", 0.5)
        return (rng.random((4, n, n, n)) < fill).astype(np.uint8)
    out = np.empty((4, n, n, n), dtype=np.uint8)
    for idx, name in enumerate(("I1", "I2", "I3", "IV")):
        frac = _frac_points(n, DOF_OFFSETS[name])
        cart = frac @ A.T
        out[idx] = contains(kind, cart, A, params).astype(np.uint8)
    return out


# --------------------------------------------------------------------------------------
# Seeded vectors
# --------------------------------------------------------------------------------------


def random_block(n: int, ncols: int, seed: int, kind: str = "white") -> np.ndarray:
    """Seeded complex block, C-contiguous (ncols, 3 n^3) (= column-major, ld = 3 n^3).

    white:  i.i.d. complex Gaussian entries.
    smooth: Fourier-space block supported on modes with |m_i| <= 2 (wrapped), Gaussian there.
    """
    rng = np.random.default_rng(seed)
    m = 3 * n ** 3
    x = rng.standard_normal((ncols, m)) + 1j * rng.standard_normal((ncols, m))
    if kind == "smooth":
        f = np.minimum(np.arange(n), n - np.arange(n))
        keep = (f[:, None, None] <= 2) & (f[None, :, None] <= 2) & (f[None, None, :] <= 2)
        keep = np.broadcast_to(keep, (3, n, n, n)).reshape(-1)
        x[:, ~keep] = 0
    return np.ascontiguousarray(x)


@dataclass(frozen=True)
class Workload:
    """A named synthetic configuration (BASELINE.json configs)."""
    name: str
    lattice: str
    geometry: str
    eps: str
    n: int
    nev: int
    segments: int

    def eps1(self) -> np.ndarray:
        return {"vacuum": np.eye(3, dtype=np.complex128),
                "iso13": eps_isotropic(13.0),
                "pc13": eps_pseudochiral(13.0, 0.875),
                "iso16": eps_isotropic(16.0),
                "pc16": eps_pseudochiral(16.0, 0.875)}[self.eps]

    def A(self) -> np.ndarray:
        return lattice(self.lattice)

    def masks(self) -> np.ndarray:
        return make_masks(self.geometry, self.A(), self.n)

    def kpoints(self) -> np.ndarray:
        if self.name == "C1":
            return np.array([[PI, PI, PI], [PI / 7, 3 * PI / 5, 4 * PI / 13]])
        return kpath(self.lattice, self.segments)


WORKLOADS = {
    "C1": Workload("C1", "sc", "vacuum", "vacuum", 8, 6, 1),
    "C2": Workload("C2", "sc", "sphere", "iso13", 32, 10, 8),
    "C3": Workload("C3", "sc", "sc_curv", "pc13", 64, 10, 8),
    "C4": Workload("C4", "fcc", "fcc_diamond", "pc13", 128, 10, 8),
    "C5": Workload("C5", "fcc", "fcc_diamond", "pc13", 192, 20, 32),
}
