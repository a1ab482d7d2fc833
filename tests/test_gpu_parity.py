"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded inputs.

Bars (BASELINE.json north_star): operator apply relative error <= 1e-12 per column (2-norm),
eigenvalues relative error <= 1e-8.  Sub-steps (FFT, M_eps, K_P^{-1}) are held to 1e-13/1e-14.
"""
import math

import numpy as np
import pytest

import synth
from oracle import pc_oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
PI = math.pi


@pytest.fixture(scope="module")
def api():
    from paper_2511_17107_b200 import api as a
    return a


def to_dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda")


def relerr_cols(got, ref):
    num = np.linalg.norm(got - ref, axis=-1)
    den = np.linalg.norm(ref, axis=-1)
    return float(np.max(num / den))


# ------------------------------------------------------------------------------------- FFT
@pytest.mark.parametrize("n", [4, 6, 8, 10, 12, 16, 20, 24, 32, 40, 48, 64, 80, 96, 100, 120, 128, 160, 192, 240, 256])
def test_fft3_matches_paper_F3(api, n):
    ctx = api.pc_create(np.eye(3), n, np.eye(3), np.zeros((4, n, n, n), np.uint8))
    nc = 2 if n <= 128 else 1
    x = synth.random_block(n, nc, seed=n)
    X = to_dev(x)
    Y = torch.empty_like(X)
    api.pc_fft3(ctx, X, Y, api.PC_FFT_TO_FOURIER)
    ref = np.stack([O.fft3_real_to_fourier(x[c], n) for c in range(nc)])
    assert relerr_cols(Y.cpu().numpy(), ref) <= 1e-13
    Z = torch.empty_like(X)
    api.pc_fft3(ctx, Y, Z, api.PC_FFT_TO_REAL)
    assert relerr_cols(Z.cpu().numpy(), x) <= 1e-13


# ------------------------------------------------------------------------------------- M_eps
@pytest.mark.parametrize("n", [4, 6, 8, 16])
@pytest.mark.parametrize("eps,mode", [("pc", "crossdof"), ("sdd", "crossdof"), ("ext", "crossdof"),
                                      ("sdd", "trivial"), ("pc", "trivial"), ("diag", "diagonal")])
def test_eps_stencil_matches_oracle(api, n, eps, mode):
    e = {"pc": synth.eps_pseudochiral(), "sdd": synth.eps_sdd(), "ext": synth.eps_extreme(),
         "diag": np.diag([0.2, 0.5, 0.9]).astype(complex)}[eps]
    masks = synth.make_masks("random", np.eye(3), n, seed=7 * n)
    ctx = api.pc_create(np.eye(3), n, e, masks, eps_mode=mode)
    x = synth.random_block(n, 3, seed=1)
    Y = torch.empty(3, 3 * n ** 3, dtype=torch.complex128, device="cuda")
    api.pc_apply_eps(ctx, to_dev(x), Y)
    M = O.permittivity_matrix(e, masks, mode)
    ref = (M @ x.T).T
    assert relerr_cols(Y.cpu().numpy(), ref) <= 1e-14


# ------------------------------------------------------------------------------------- K_P^{-1}
@pytest.mark.parametrize("lat,n,k", [("sc", 8, (0.3, -1.1, 2.0)), ("fcc", 12, (PI, PI, PI)), ("sc", 6, (0, 0, 0)),
                                     ("bcc", 8, (0.05, 0.02, -0.01)), ("fcc", 16, (0, 2 * PI, 0))])
def test_precond_matches_oracle(api, lat, n, k):
    A = synth.lattice(lat)
    ctx = api.pc_create(A, n, np.eye(3), np.zeros((4, n, n, n), np.uint8))
    r = synth.random_block(n, 2, seed=3)
    P = torch.empty(2, 3 * n ** 3, dtype=torch.complex128, device="cuda")
    api.pc_precond(ctx, k, to_dev(r), P)
    gamma = O.gamma_rule(k)
    assert abs(api.pc_gamma(ctx, k) - gamma) <= 1e-12 * gamma
    ref = O.precond_fourier(n, np.array(k), A, gamma, r)
    assert relerr_cols(P.cpu().numpy(), ref) <= 1e-12


PRECOND_EPS_CASES = [
    ("fcc", "fcc_diamond", "pc", "crossdof", 8, (PI, PI, PI)),
    ("sc", "sphere", "iso", "crossdof", 12, (0.0, 0.0, 0.0)),
    ("sc", "random", "sdd", "crossdof", 16, (0.3, -1.2, 2.5)),
    ("bcc", "random", "pc", "trivial", 10, (2 * PI, 0, 0)),
    ("fcc", "fcc_diamond", "pc", "crossdof", 128, (PI / 2, 2 * PI, PI / 2)),
]


@pytest.mark.parametrize("lat,geo,eps,mode,n,k", PRECOND_EPS_CASES)
def test_precond_eps_matches_oracle(api, lat, geo, eps, mode, n, k):
    """Option precond = 1 (eps-weighted preconditioner, reading R16): pc_precond against the oracle's
    explicit per-mode formula, including k = 0 (zero mode -> 0) and the n = 128 bench grid."""
    A = synth.lattice(lat)
    e = _eps(eps)
    masks = synth.make_masks(geo, A, n, seed=11)
    ctx = api.pc_create(A, n, e, masks, eps_mode=mode)
    api.pc_set_option(ctx, "precond", 1)
    nc = 1 if n >= 64 else 2
    r = synth.random_block(n, nc, seed=21)
    P = torch.empty(nc, 3 * n ** 3, dtype=torch.complex128, device="cuda")
    api.pc_precond(ctx, k, to_dev(r), P)
    ref = O.precond_eps_fourier(n, np.array(k), A, O.gamma_rule(np.array(k)), e, masks, mode, r)
    assert relerr_cols(P.cpu().numpy(), ref) <= 1e-12


# ------------------------------------------------------------------------------------- apply
APPLY_CASES = [
    ("sc", "random", "pc", "crossdof", 4, (PI, PI, PI)),
    ("sc", "random", "sdd", "crossdof", 6, (0.3, -1.2, 2.5)),
    ("fcc", "random", "pc", "crossdof", 8, (0.7, 1.9, -2.2)),
    ("bcc", "random", "sdd", "crossdof", 8, (2 * PI, 0, 0)),
    ("sc", "random", "pc", "trivial", 8, (0.1, 0.05, 0.0)),
    ("fcc", "random", "ext", "crossdof", 10, (0.0, 0.0, 0.0)),
    ("sc", "sphere", "iso", "crossdof", 16, (PI / 2, 0.0, 0.0)),
    ("sc", "sc_curv", "pc", "crossdof", 24, (PI, PI, 0)),
    ("fcc", "fcc_diamond", "pc", "crossdof", 32, (PI, PI, PI)),
    ("fcc", "fcc_diamond", "pc", "crossdof", 20, (PI / 2, 2 * PI, PI / 2)),
]


def _eps(name):
    return {"pc": synth.eps_pseudochiral(), "sdd": synth.eps_sdd(), "ext": synth.eps_extreme(),
            "iso": synth.eps_isotropic(13.0)}[name]


@pytest.mark.parametrize("lat,geo,eps,mode,n,k", APPLY_CASES)
def test_apply_fourier_matches_oracle(api, lat, geo, eps, mode, n, k):
    A = synth.lattice(lat)
    e = _eps(eps)
    masks = synth.make_masks(geo, A, n, seed=11)
    ctx = api.pc_create(A, n, e, masks, eps_mode=mode)
    x = np.concatenate([synth.random_block(n, 2, seed=5), synth.random_block(n, 1, seed=6, kind="smooth")])
    Y = torch.empty(3, 3 * n ** 3, dtype=torch.complex128, device="cuda")
    api.pc_apply(ctx, k, to_dev(x), Y)
    op = O.PenalizedOperator(n, np.array(k), A, e, masks, mode)
    ref = op.apply_fourier(x)
    assert relerr_cols(Y.cpu().numpy(), ref) <= 1e-12


@pytest.mark.parametrize("lat,n,k", [("sc", 8, (0.4, 0.1, -0.3)), ("fcc", 12, (PI, PI, PI))])
def test_apply_real_space_matches_oracle(api, lat, n, k):
    A = synth.lattice(lat)
    e = synth.eps_sdd()
    masks = synth.make_masks("random", A, n, seed=2)
    ctx = api.pc_create(A, n, e, masks)
    H = synth.random_block(n, 2, seed=9)
    Y = torch.empty(2, 3 * n ** 3, dtype=torch.complex128, device="cuda")
    api.pc_apply(ctx, k, to_dev(H), Y, space=api.PC_SPACE_REAL)
    op = O.PenalizedOperator(n, np.array(k), A, e, masks)
    ref = np.stack([op.apply_real(H[c]) for c in range(2)])
    assert relerr_cols(Y.cpu().numpy(), ref) <= 1e-12


@pytest.mark.parametrize("lat,geo,n", [("fcc", "fcc_diamond", 16), ("sc", "sc_curv", 12)])
def test_apply_and_precond_multi_k_match_oracle(api, lat, geo, n):
    """several Bloch vectors in one launch (per-column symbol tables, penalties and
    thresholds), including k = 0 and a k with ||k|| < 1 (gamma = 4 pi^2/||k||^2), against the
    oracle's apply and K_P^{-1} for each column's own k (<= 1e-12)."""
    A = synth.lattice(lat)
    e = synth.eps_pseudochiral()
    masks = synth.make_masks(geo, A, n)
    kp = np.array([[PI, PI, PI], [0.0, 0.0, 0.0], [0.3, -0.2, 0.5], [1.1, 2.0, -0.4]])
    kcol = [0, 1, 2, 3, 2, 0, 3]
    ctx = api.pc_create(A, n, e, masks)
    x = synth.random_block(n, len(kcol), seed=17)
    X = to_dev(x)
    Y = torch.empty_like(X)
    P = torch.empty_like(X)
    api.pc_apply_multi(ctx, kp, kcol, X, Y)
    api.pc_precond_multi(ctx, kp, kcol, X, P)
    Yh, Ph = Y.cpu().numpy(), P.cpu().numpy()
    for j, ki in enumerate(kcol):
        op = O.PenalizedOperator(n, kp[ki], A, e, masks)
        assert relerr_cols(Yh[j:j + 1], op.apply_fourier(x[j:j + 1])) <= 1e-12
        ref = O.precond_fourier(n, kp[ki], A, op.gamma, x[j:j + 1])
        assert relerr_cols(Ph[j:j + 1], ref) <= 1e-12
    # same result as one-k launches
    Y1 = torch.empty_like(X)
    for j, ki in enumerate(kcol):
        api.pc_apply(ctx, kp[ki], X[j:j + 1], Y1[j:j + 1])
    assert relerr_cols(Y1.cpu().numpy(), Yh) <= 1e-14


def test_apply_gamma_override_and_ld(api):
    """Strided blocks (ld > 3N^3) and the gamma override path."""
    n, A, k = 8, synth.lattice("sc"), (0.2, 0.3, 0.1)
    e = synth.eps_pseudochiral()
    masks = synth.make_masks("random", A, n, seed=4)
    ctx = api.pc_create(A, n, e, masks, gamma_override=2.5)
    x = synth.random_block(n, 2, seed=8)
    big = torch.zeros(2, 3 * n ** 3 + 64, dtype=torch.complex128, device="cuda")
    big[:, : 3 * n ** 3] = to_dev(x)
    out = torch.zeros_like(big)
    api.pc_apply(ctx, k, big[:, : 3 * n ** 3], out[:, : 3 * n ** 3])
    ref = O.PenalizedOperator(n, np.array(k), A, e, masks, gamma=2.5).apply_fourier(x)
    assert relerr_cols(out[:, : 3 * n ** 3].cpu().numpy(), ref) <= 1e-12
    assert torch.all(out[:, 3 * n ** 3:] == 0)


# ------------------------------------------------------------------- full size (bench config)
@pytest.mark.parametrize("plane", [1, 0])
def test_apply_full_size_n128_fcc_pseudochiral(api, plane):
    """BASELINE config C4 at full size, the bench's launch configuration (a 15-column block), with the
    fused cluster plane pass (plane.cu) and with the three-pass middle section."""
    W = synth.WORKLOADS["C4"]
    n, A, e, masks = W.n, W.A(), W.eps1(), W.masks()
    k = np.array([PI, PI, PI])
    ctx = api.pc_create(A, n, e, masks)
    api.pc_set_option(ctx, "plane_fuse", plane)
    x = np.concatenate([synth.random_block(n, 1, seed=21), synth.random_block(n, 1, seed=22, kind="smooth")])
    X = torch.zeros(15, 3 * n ** 3, dtype=torch.complex128, device="cuda")
    X[:2] = to_dev(x)
    X[2:] = torch.randn(13, 3 * n ** 3, dtype=torch.complex128, device="cuda")
    Y = torch.empty_like(X)
    api.pc_apply(ctx, k, X, Y)
    op = O.PenalizedOperator(n, k, A, e, masks)
    ref = op.apply_fourier(x)
    assert relerr_cols(Y[:2].cpu().numpy(), ref) <= 1e-12


def test_apply_full_size_n192_c5(api):
    """BASELINE config C5 (FCC diamond pseudochiral, n = 192: the 16 x 12 radix plan) at full size, a
    26-column block (C5's b = nev + guard) with two oracle columns (white and smooth), <= 1e-12."""
    W = synth.WORKLOADS["C5"]
    n, A, e, masks = W.n, W.A(), W.eps1(), W.masks()
    k = np.array([PI / 2, 2 * PI, PI / 2])
    ctx = api.pc_create(A, n, e, masks)
    x = np.concatenate([synth.random_block(n, 1, seed=31), synth.random_block(n, 1, seed=32, kind="smooth")])
    X = torch.randn(26, 3 * n ** 3, dtype=torch.complex128, device="cuda")
    X[:2] = to_dev(x)
    Y = torch.empty_like(X)
    api.pc_apply(ctx, k, X, Y)
    torch.cuda.synchronize()
    got = Y[:2].cpu().numpy()
    del X, Y
    op = O.PenalizedOperator(n, k, A, e, masks)
    assert relerr_cols(got, op.apply_fourier(x)) <= 1e-12


@pytest.mark.parametrize("plane", [1])
@pytest.mark.parametrize("mode,eps,geo", [("diagonal", "iso", "sphere"), ("trivial", "sdd", "random"),
                                           ("crossdof", "pc", "random")])
def test_apply_plane_pass_n128_modes(api, mode, eps, geo, plane):
    """The cluster plane passes (n = 128, plane2.cu: 16-CTA clusters) in every mode they
    serve against the oracle (one white column), and against the three-pass middle section on a
    4-column block (<= 1e-13)."""
    n = 128
    A = synth.lattice("sc")
    e = {"pc": synth.eps_pseudochiral(), "sdd": synth.eps_sdd(), "iso": synth.eps_isotropic(13.0)}[eps]
    masks = synth.make_masks(geo, A, n, seed=5)
    k = np.array([0.3, -1.2, 2.0])
    ctx = api.pc_create(A, n, e, masks, eps_mode=mode)
    X = torch.randn(4, 3 * n ** 3, dtype=torch.complex128, device="cuda")
    Y1, Y0 = torch.empty_like(X), torch.empty_like(X)
    api.pc_set_option(ctx, "plane_fuse", plane)
    api.pc_apply(ctx, k, X, Y1)
    api.pc_set_option(ctx, "plane_fuse", 0)
    api.pc_apply(ctx, k, X, Y0)
    assert relerr_cols(Y1.cpu().numpy(), Y0.cpu().numpy()) <= 1e-13
    op = O.PenalizedOperator(n, k, A, e, masks, mode)
    ref = op.apply_fourier(X[:1].cpu().numpy())
    assert relerr_cols(Y1[:1].cpu().numpy(), ref) <= 1e-12


def _kappa2_closed(n, k, A):
    """|kappa(m)|^2 from the symbols lambda_1 = (1 - e^{-i theta})/h, lambda_0 = (1 + e^{-i theta})/2."""
    h = 1.0 / n
    th = 2 * PI * np.arange(n) / n
    l1 = (1 - np.exp(-1j * th)) / h
    l0 = (1 + np.exp(-1j * th)) / 2
    B = np.linalg.inv(A)
    grids = [l1[None, None, :], l1[None, :, None], l1[:, None, None]]
    g0 = [l0[None, None, :], l0[None, :, None], l0[:, None, None]]
    tot = 0
    for i in range(3):
        kap = sum(B[j, i] * grids[j] for j in range(3)) + 1j * k[i] * g0[i]
        tot = tot + np.abs(kap) ** 2
    return np.broadcast_to(tot, (n, n, n))


@pytest.mark.parametrize("lat,n", [("sc", 128), ("fcc", 128), ("fcc", 192)])
def test_identity_selftest_full_size(api, lat, n):
    """M = I, gamma = 1: A_c A_c^H + B^H B = diag(L, L, L), so the apply is
    multiplication by |kappa(m)|^2 per mode -- an oracle-free check at the full sizes."""
    A = synth.lattice(lat)
    k = np.array([0.9, -2.1, PI])
    ctx = api.pc_create(A, n, np.eye(3), np.zeros((4, n, n, n), np.uint8), gamma_override=1.0)
    X = torch.randn(2, 3 * n ** 3, dtype=torch.complex128, device="cuda")
    Y = torch.empty_like(X)
    api.pc_apply(ctx, k, X, Y)
    k2 = torch.from_numpy(np.tile(_kappa2_closed(n, k, A).reshape(-1), 3)).to("cuda")
    ref = X * k2[None, :]
    err = (torch.linalg.vector_norm(Y - ref, dim=1) / torch.linalg.vector_norm(ref, dim=1)).max().item()
    assert err <= 1e-12


# ------------------------------------------------------------------------------------- Jacobi
@pytest.mark.parametrize("n", [1, 2, 5, 16, 36, 45, 75, 80])
def test_device_jacobi_eigh(api, n):
    """The Rayleigh-Ritz eigensolver (one-CTA cyclic Jacobi) against numpy on Hermitian matrices with
    spectra over 7 decades, a degenerate cluster and a diagonal matrix."""
    rng = np.random.default_rng(n)
    M = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    M = M + M.conj().T
    # widen the spectrum to mimic H (1 .. 1e7)
    Q, _ = np.linalg.qr(M)
    M = Q @ np.diag(np.logspace(0, 7, n)) @ Q.conj().T if n > 3 else M
    M = 0.5 * (M + M.conj().T)
    w, V, sw = api.pc_debug_heevj(M)
    wr = np.linalg.eigvalsh(M)
    assert np.allclose(w, wr, rtol=1e-12, atol=1e-12 * np.abs(wr).max())
    assert np.allclose(V.conj().T @ V, np.eye(n), atol=1e-12)
    assert np.linalg.norm(M @ V - V * w[None, :]) <= 1e-12 * np.linalg.norm(M)
    # a degenerate cluster (as at symmetry points) and a diagonal matrix (all rotations trivial)
    if n >= 5:
        D = np.diag(np.r_[np.full(3, 2.0), np.arange(n - 3) + 3.0]).astype(complex)
        Qr, _ = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
        for Mx in (Qr @ D @ Qr.conj().T, D):
            Mx = 0.5 * (Mx + Mx.conj().T)
            w2, V2, _ = api.pc_debug_heevj(Mx)
            assert np.allclose(w2, np.linalg.eigvalsh(Mx), atol=1e-12 * n)
            assert np.allclose(V2.conj().T @ V2, np.eye(n), atol=1e-12)


@pytest.mark.parametrize("eps,mode,n", [("pc", "crossdof", 16), ("iso", "crossdof", 12), ("sdd", "trivial", 8),
                                        ("pc", "crossdof", 128)])
def test_fused_xex_pipeline_matches_unfused(api, eps, mode, n):
    """The fused x-DFT + M_eps + x-DFT pass (z-plane-local media) against the 7-pass pipeline and the oracle."""
    A = synth.lattice("fcc")
    e = _eps(eps)
    masks = synth.make_masks("fcc_diamond" if n > 16 else "random", A, n, seed=13)
    ctx = api.pc_create(A, n, e, masks, eps_mode=mode)
    k = (PI, 0.4, -1.3)
    X = torch.randn(3, 3 * n ** 3, dtype=torch.complex128, device="cuda")
    Y1 = torch.empty_like(X)
    Y0 = torch.empty_like(X)
    api.pc_apply(ctx, k, X, Y1)
    api.pc_set_option(ctx, "fuse_xex", 0)
    api.pc_apply(ctx, k, X, Y0)
    err = (torch.linalg.vector_norm(Y1 - Y0, dim=1) / torch.linalg.vector_norm(Y0, dim=1)).max().item()
    assert err <= 1e-13
    if n <= 16:
        op = O.PenalizedOperator(n, np.array(k), A, e, masks, mode)
        assert relerr_cols(Y1.cpu().numpy(), op.apply_fourier(X.cpu().numpy())) <= 1e-12


@pytest.mark.parametrize("eps,n", [("sdd", 8), ("pc", 12), ("pc", 64)])
def test_library_composition_baseline_matches(api, eps, n):
    """The cuFFT + elementwise comparison arm (tools/library_apply.py, timed by bench.py) computes the
    same operator: against the oracle at small n and against pc_apply at n = 64."""
    import os
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    from library_apply import LibraryApply
    A = synth.lattice("fcc")
    e = _eps(eps)
    masks = synth.make_masks("random" if n <= 12 else "fcc_diamond", A, n, seed=5)
    k = np.array([0.7, -PI / 3, 1.9])
    ctx = api.pc_create(A, n, e, masks)
    X = torch.randn(2, 3 * n ** 3, dtype=torch.complex128, device="cuda")
    Y = torch.empty_like(X)
    api.pc_apply(ctx, k, X, Y)
    L = LibraryApply(n, A, k, e, masks, api.pc_gamma(ctx, k), "cuda")
    Yl = L(X)
    err = (torch.linalg.vector_norm(Yl - Y, dim=1) / torch.linalg.vector_norm(Y, dim=1)).max().item()
    assert err <= 1e-12
    if n <= 12:
        op = O.PenalizedOperator(n, k, A, e, masks, "crossdof")
        assert relerr_cols(Yl.cpu().numpy(), op.apply_fourier(X.cpu().numpy())) <= 1e-12
