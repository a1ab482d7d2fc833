"""Pins of the CPU oracle against what PAPER.md and mathematics fix (no GPU needed).

Each test names the passage it pins.  None of them re-calls the oracle routine it checks
with the same formula: literal matrices typed from the paper, explicit stencil loops
transcribed from the paper's component formulas, theorems (Lemma 2.1, Props 2.2/2.4,
Lemma 2.3, Props 3.4-3.8) and closed-form spectra.
"""
import math

import numpy as np
import pytest

import synth
from oracle import pc_oracle as O

PI = math.pi
RNG = np.random.default_rng(12345)


def _roll(a, shift, axis):
    return np.roll(a, shift, axis=axis)


# ---------------------------------------------------------------- P:182-193 literal matrices
def test_circulants_literal_P183():
    n = 4
    D1 = 4.0 * np.array([[1, 0, 0, -1], [-1, 1, 0, 0], [0, -1, 1, 0], [0, 0, -1, 1]])
    D0 = 0.5 * np.array([[1, 0, 0, 1], [1, 1, 0, 0], [0, 1, 1, 0], [0, 0, 1, 1]])
    assert np.array_equal(O.circulant_D1(n).toarray(), D1)
    assert np.array_equal(O.circulant_D0(n).toarray(), D0)


# ---------------------------------------------------------------- Lemma 2.1
def test_dft_convention_P274():
    F = O.dft_matrix(4)
    assert abs(F[1, 1] - 1j / 2) < 1e-15           # w = exp(+2 pi i / N)
    assert np.allclose(F @ F.conj().T, np.eye(4), atol=1e-14)


@pytest.mark.parametrize("n", [4, 5, 7])
def test_lemma21_circulant_diagonalisation(n):
    c = RNG.standard_normal(n) + 1j * RNG.standard_normal(n)
    C = np.array([[c[(j - i) % n] for j in range(n)] for i in range(n)])  # first row c
    lam = O.circulant_symbols(c)
    F = O.dft_matrix(n)
    assert np.allclose(F @ np.diag(lam) @ F.conj().T, C, atol=1e-12)


def test_D0_symbols_paper_convention_N4():
    # under P:274 the D0 symbols at N=4 are (1, (1-i)/2, 0, (1+i)/2)
    # (SPEC S:188 prints the conjugate convention).
    _, l0 = O.symbols_1d(4)
    assert np.allclose(l0, [1, 0.5 - 0.5j, 0, 0.5 + 0.5j], atol=1e-15)


def test_fft3_is_paper_F3():
    # x = F3^H H with F3 = F (x) F (x) F per component.
    n = 3
    F = O.dft_matrix(n)
    F3 = np.kron(np.kron(F, F), F)
    H = RNG.standard_normal(3 * n ** 3) + 1j * RNG.standard_normal(3 * n ** 3)
    x = O.fft3_real_to_fourier(H, n)
    for c in range(3):
        sl = slice(c * n ** 3, (c + 1) * n ** 3)
        assert np.allclose(x[sl], F3.conj().T @ H[sl], atol=1e-13)
    assert np.allclose(O.fft3_fourier_to_real(x, n), H, atol=1e-13)


# ---------------------------------------------------------------- stencils P:158-179
def _split(v, n):
    return [v[c * n ** 3:(c + 1) * n ** 3].reshape(n, n, n) for c in range(3)]


@pytest.mark.parametrize("n", [4, 5])
def test_curl_stencil_P160(n):
    """Component formulas of P:160-165 (x = axis 2, y = axis 1, z = axis 0 of [z][y][x]),
    with the P:163 sign typo read per the matrix form (reading R1)."""
    h = 1.0 / n
    k = RNG.uniform(-PI, PI, 3)
    E = RNG.standard_normal(3 * n ** 3) + 1j * RNG.standard_normal(3 * n ** 3)
    E1, E2, E3 = _split(E, n)
    X, Y, Z = 2, 1, 0
    m = lambda a, ax: _roll(a, 1, ax)  # value at index-1
    F1 = (E3 - m(E3, Y)) / h - (E2 - m(E2, Z)) / h + 1j * (k[1] * (m(E3, Y) + E3) / 2 - k[2] * (m(E2, Z) + E2) / 2)
    F2 = (E1 - m(E1, Z)) / h - (E3 - m(E3, X)) / h + 1j * (k[2] * (m(E1, Z) + E1) / 2 - k[0] * (m(E3, X) + E3) / 2)
    F3 = (E2 - m(E2, X)) / h - (E1 - m(E1, Y)) / h + 1j * (k[0] * (m(E2, X) + E2) / 2 - k[1] * (m(E1, Y) + E1) / 2)
    ref = np.concatenate([F1.ravel(), F2.ravel(), F3.ravel()])
    got = O.curl_matrix(n, k, np.eye(3)) @ E
    assert np.allclose(got, ref, atol=1e-12)


def test_div_stencil_P169():
    n = 5
    h = 1.0 / n
    k = RNG.uniform(-PI, PI, 3)
    H = RNG.standard_normal(3 * n ** 3) + 1j * RNG.standard_normal(3 * n ** 3)
    H1, H2, H3 = _split(H, n)
    m = lambda a, ax: _roll(a, 1, ax)
    ref = ((H1 - m(H1, 2)) + (H2 - m(H2, 1)) + (H3 - m(H3, 0))) / h + 1j * (
        k[0] * (m(H1, 2) + H1) / 2 + k[1] * (m(H2, 1) + H2) / 2 + k[2] * (m(H3, 0) + H3) / 2)
    assert np.allclose(O.div_matrix(n, k, np.eye(3)) @ H, ref.ravel(), atol=1e-12)


@pytest.mark.parametrize("n", [4, 5])
def test_crossdof_templates_P647(n):
    """T_ij as 4-point averages of the neighbouring staggered DoFs (reading R4/R5):
    (T12 E2)(i,j,k) = 1/4 sum_{a in {-1,0}, b in {0,1}} E2(i+a, j+b, k), etc."""
    T12, T13, T23 = O.transfer_T(n)
    v = RNG.standard_normal((n, n, n)) + 1j * RNG.standard_normal((n, n, n))
    def sh(a, dx=0, dy=0, dz=0):  # value at (i+dx, j+dy, k+dz)
        return np.roll(a, (-dz, -dy, -dx), axis=(0, 1, 2))
    t12 = sum(sh(v, a, b, 0) for a in (-1, 0) for b in (0, 1)) / 4
    t13 = sum(sh(v, a, 0, c) for a in (-1, 0) for c in (0, 1)) / 4
    t23 = sum(sh(v, 0, b, c) for b in (-1, 0) for c in (0, 1)) / 4
    assert np.allclose(T12 @ v.ravel(), t12.ravel(), atol=1e-14)
    assert np.allclose(T13 @ v.ravel(), t13.ravel(), atol=1e-14)
    assert np.allclose(T23 @ v.ravel(), t23.ravel(), atol=1e-14)
    # transposes mirror the offsets
    t12t = sum(sh(v, a, b, 0) for a in (0, 1) for b in (-1, 0)) / 4
    assert np.allclose(T12.T @ v.ravel(), t12t.ravel(), atol=1e-14)


# ---------------------------------------------------------------- Prop 2.2
@pytest.mark.parametrize("lat", ["sc", "fcc", "bcc"])
def test_BA_zero(lat):
    n = 5
    k = RNG.uniform(-PI, PI, 3)
    A = synth.lattice(lat)
    BA = O.div_matrix(n, k, A) @ O.curl_matrix(n, k, A)
    assert abs(BA).max() <= 1e-10 * n * n


# ---------------------------------------------------------------- Lemma 2.3
def test_lemma23_block_laplacian():
    n = 4
    k = RNG.uniform(-PI, PI, 3)
    Ac = O.curl_matrix(n, k, np.eye(3)).toarray()
    B = O.div_matrix(n, k, np.eye(3)).toarray()
    D = O.shifted_blocks(n, k, np.eye(3))
    L = sum((Di.conj().T @ Di).toarray() for Di in D)
    lhs = Ac @ Ac.conj().T + B.conj().T @ B
    Z = np.zeros_like(L)
    rhs = np.block([[L, Z, Z], [Z, L, Z], [Z, Z, L]])
    assert np.allclose(lhs, rhs, atol=1e-10)
    assert np.allclose(L, B @ B.conj().T, atol=1e-10)


@pytest.mark.parametrize("n,kk", [(8, 0.7), (8, PI), (6, -2.1), (9, 1.3)])
def test_mu_closed_form_P394(n, kk):
    h = 1.0 / n
    K = (O.circulant_D1(n) + 1j * kk * O.circulant_D0(n)).toarray()
    ev = np.sort(np.linalg.eigvalsh(K.conj().T @ K))
    phi = math.atan2(4 * kk * h, 4 - kk * kk * h * h)
    mu = np.sort([(2 / h ** 2 + kk ** 2 / 2) * (1 - math.cos(phi + 2 * j * PI * h)) for j in range(1, n + 1)])
    assert np.allclose(ev, mu, rtol=1e-12, atol=1e-10)
    assert abs(mu.min() - kk * kk) <= 1e-10 * max(1, kk * kk)


@pytest.mark.parametrize("n", [6, 8])
def test_lambda_min_L_equals_k2_P379(n):
    k = RNG.uniform(-PI, PI, 3)
    D = O.shifted_blocks(n, k, np.eye(3))
    L = sum((Di.conj().T @ Di).toarray() for Di in D)
    assert abs(np.linalg.eigvalsh(L).min() - k @ k) <= 1e-9


# ---------------------------------------------------------------- Prop 2.4
@pytest.mark.parametrize("lat", ["sc", "fcc"])
def test_null_space_k0_P417(lat):
    n = 4
    A = synth.lattice(lat)
    masks = synth.make_masks("random", A, n, seed=3)
    op = O.PenalizedOperator(n, np.zeros(3), A, synth.eps_pseudochiral(), masks)
    w = np.linalg.eigvalsh(op.dense())
    assert np.sum(np.abs(w) < 1e-9) == 3 and w[3] > 1e-3
    for c in range(3):
        o = np.zeros(op.dim)
        o[c * n ** 3:(c + 1) * n ** 3] = 1.0
        assert np.linalg.norm(op.apply_real(o)) < 1e-10
    op2 = O.PenalizedOperator(n, np.array([0.3, -0.2, 0.5]), A, synth.eps_pseudochiral(), masks)
    assert np.linalg.eigvalsh(op2.dense()).min() > 1e-6


def test_gamma_rule_P457():
    assert O.gamma_rule([0, 0, 0]) == 4 * PI ** 2
    assert O.gamma_rule([PI, PI, PI]) == 4 * PI ** 2
    assert abs(O.gamma_rule([0.1, 0, 0]) - 400 * PI ** 2) < 1e-9
    assert abs(O.gamma_rule([0.3, 0.4, 0]) - 4 * PI ** 2 / 0.25) < 1e-9


# ---------------------------------------------------------------- Prop 2.2 spectrum union
@pytest.mark.parametrize("lat", ["sc", "fcc"])
def test_spectrum_union_P295(lat):
    n = 4
    A = synth.lattice(lat)
    k = np.array([0.4, -0.9, 1.7])
    masks = synth.make_masks("random", A, n, seed=5)
    gamma = 3.7
    op = O.PenalizedOperator(n, k, A, synth.eps_pseudochiral(), masks, gamma=gamma)
    Ac, M, B = op.Ac.toarray(), op.M.toarray(), op.B.toarray()
    full = np.linalg.eigvalsh(op.dense())
    a = np.linalg.eigvalsh(Ac @ M @ Ac.conj().T)
    b = np.linalg.eigvalsh(B.conj().T @ B)
    thr = 1e-8 * full.max()
    union = np.sort(np.concatenate([a[a > thr], gamma * b[b > thr]]))
    pos = full[full > thr]
    assert union.size == pos.size
    assert np.allclose(pos, union, rtol=1e-10, atol=1e-9)


# ---------------------------------------------------------------- vacuum closed form
def _vacuum_closed_form(n, k, gamma):
    """{|kappa|^2 (x2), gamma |kappa|^2} per mode with |kappa(m)|^2 = sum_i mu^{(i)}_{m_i}
    from P:394 (A = I; spectrum of diag(L,L,L) split by the penalty)."""
    h = 1.0 / n
    mus = []
    for ki in k:
        phi = math.atan2(4 * ki * h, 4 - ki * ki * h * h)
        mus.append(np.array([(2 / h ** 2 + ki ** 2 / 2) * (1 - math.cos(phi + 2 * j * PI * h)) for j in range(n)]))
    tot = (mus[0][None, None, :] + mus[1][None, :, None] + mus[2][:, None, None]).ravel()
    return np.sort(np.concatenate([tot, tot, gamma * tot]))


@pytest.mark.parametrize("k", [(PI, PI, PI), (0.3, -1.2, 2.5), (0.0, 0.0, 0.0)])
def test_vacuum_closed_form(k):
    n = 4
    k = np.array(k)
    op = O.PenalizedOperator(n, k, np.eye(3), np.eye(3), synth.make_masks("vacuum", np.eye(3), n))
    w = np.linalg.eigvalsh(op.dense())
    ref = _vacuum_closed_form(n, k, op.gamma)
    assert np.allclose(w, ref, rtol=1e-11, atol=1e-9)


def test_vacuum_golden_n8():
    rows = {}
    for line in open(__file__.replace("test_oracle_pins.py", "golden/c1_vacuum_n8.txt")):
        if line.startswith("#") or not line.strip():
            continue
        name, *vals = line.split()
        rows[name] = np.array([float(v) for v in vals])
    masks = synth.make_masks("vacuum", np.eye(3), 8)
    for name, k in (("k_a", (PI, PI, PI)), ("k_b", (PI / 7, 3 * PI / 5, 4 * PI / 13))):
        op = O.PenalizedOperator(8, np.array(k), np.eye(3), np.eye(3), masks)
        w = O.eigs_dense(op, 6)
        assert np.allclose(w, rows[name], rtol=1e-11)


# ---------------------------------------------------------------- homogeneous closed form
def _homog_closed_form(n, k, A, eps1, gamma):
    """FULL masks: S_ij = T_ij circulant; per mode the operator is
    K_A Mhat K_A^H + gamma conj(kappa) kappa^T with Mhat_ij = eps_ij t_ij, t12 = l0(m1) conj l0(m2),
    t13 = l0(m1) conj l0(m3), t23 = l0(m2) conj l0(m3); symbols with
    theta = 2 pi m/N: l1 = (1 - e^{-i theta})/h, l0 = (1 + e^{-i theta})/2."""
    h = 1.0 / n
    th = 2 * PI * np.arange(n) / n
    l1 = (1 - np.exp(-1j * th)) / h
    l0 = (1 + np.exp(-1j * th)) / 2
    B = np.linalg.inv(A)
    vals = []
    for m3 in range(n):
        for m2 in range(n):
            for m1 in range(n):
                m = (m1, m2, m3)
                kap = np.array([sum(B[j, i] * l1[m[j]] for j in range(3)) + 1j * k[i] * l0[m[i]] for i in range(3)])
                KA = np.array([[0, -kap[2], kap[1]], [kap[2], 0, -kap[0]], [-kap[1], kap[0], 0]])
                t = {(0, 1): l0[m1] * np.conj(l0[m2]), (0, 2): l0[m1] * np.conj(l0[m3]), (1, 2): l0[m2] * np.conj(l0[m3])}
                Mh = np.array(eps1, dtype=complex).copy()
                for (i, j), tij in t.items():
                    Mh[i, j] = eps1[i, j] * tij
                    Mh[j, i] = np.conj(eps1[i, j]) * np.conj(tij)
                Km = KA @ Mh @ KA.conj().T + gamma * np.outer(np.conj(kap), kap)
                vals.extend(np.linalg.eigvalsh(Km))
    return np.sort(vals)


@pytest.mark.parametrize("lat,eps", [("sc", "pc"), ("fcc", "pc"), ("sc", "sdd"), ("bcc", "sdd")])
def test_homogeneous_closed_form(lat, eps):
    n = 4
    A = synth.lattice(lat)
    eps1 = synth.eps_pseudochiral() if eps == "pc" else synth.eps_sdd()
    k = np.array([1.1, -0.4, 2.2])
    op = O.PenalizedOperator(n, k, A, eps1, synth.make_masks("full", A, n))
    w = np.linalg.eigvalsh(op.dense())
    ref = _homog_closed_form(n, k, A, eps1, op.gamma)
    assert np.allclose(w, ref, rtol=1e-10, atol=1e-9)


def test_homogeneous_golden_n8():
    rows = {}
    for line in open(__file__.replace("test_oracle_pins.py", "golden/homog_n8_R.txt")):
        if line.startswith("#") or not line.strip():
            continue
        name, *vals = line.split()
        rows[name] = np.array([float(v) for v in vals])
    for lat in ("sc", "fcc"):
        A = synth.lattice(lat)
        op = O.PenalizedOperator(8, np.array([PI, PI, PI]), A, synth.eps_pseudochiral(), synth.make_masks("full", A, 8))
        w = O.eigs_dense(op, 10)
        assert np.allclose(w, rows[lat], rtol=1e-10)


# ---------------------------------------------------------------- HPD
@pytest.mark.parametrize("seed", range(4))
def test_crossdof_hpd_and_hermitian(seed):
    n = 4
    masks = synth.make_masks("random", np.eye(3), n, seed=100 + seed)
    for eps1 in (synth.eps_pseudochiral(), synth.eps_sdd(), synth.eps_pseudochiral(16.0)):
        M = O.permittivity_matrix(eps1, masks, "crossdof").toarray()
        assert np.allclose(M, M.conj().T, atol=0)
        np.linalg.cholesky(M)  # Props 3.6 / 3.8: HPD under Assumptions 1+2 or 1+3
        assert O.hpd_report(eps1)["guaranteed"]


@pytest.mark.parametrize("seed", range(3))
def test_trivial_lambda_min_bound_P755(seed):
    n = 4
    masks = synth.make_masks("random", np.eye(3), n, seed=200 + seed)
    for eps1 in (synth.eps_pseudochiral(), synth.eps_sdd()):
        M = O.permittivity_matrix(eps1, masks, "trivial").toarray()
        eh = eps1.copy()
        for i in range(3):
            eh[i, i] = min(eps1[i, i].real, 1.0)
        assert np.linalg.eigvalsh(M).min() >= np.linalg.eigvalsh(eh).min() - 1e-12


def test_S_norm_le_1_P791():
    """Prop 3.5: ||S_ij|| <= 1, on the S_ij blocks of the oracle's own M_CrossDoF
    (eps_ij = 1 off the diagonal makes the (i,j) block equal to S_ij)."""
    n = 4
    masks = synth.make_masks("random", np.eye(3), n, seed=9)
    M = O.permittivity_matrix(np.ones((3, 3), complex), masks, "crossdof").toarray()
    N3 = n ** 3
    for i, j in [(0, 1), (0, 2), (1, 2)]:
        S = M[i * N3:(i + 1) * N3, j * N3:(j + 1) * N3]
        assert abs(S).max() > 0
        assert np.linalg.norm(S, 2) <= 1 + 1e-12
        for p in (1, np.inf):
            assert np.linalg.norm(S, p) <= 1 + 1e-12


def _dof_positions(n):
    """DoF locations in units of h, 0-based index (a,b,c) = (x,y,z) (reading R6):
    E1 at (a+1/2, b+1, c+1), E2 at (a+1, b+1/2, c+1), E3 at (a+1, b+1, c+1/2).  Row order of
    a component block: flat index (c*n + b)*n + a (x fastest)."""
    c, b, a = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    base = np.stack([a.ravel(), b.ravel(), c.ravel()], axis=1).astype(float) + 1.0
    return [base - np.array(off) for off in ((0.5, 0, 0), (0, 0.5, 0), (0, 0, 0.5))]


@pytest.mark.parametrize("mode", ["diagonal", "trivial", "crossdof"])
@pytest.mark.parametrize("n", [4, 5])
def test_permittivity_entrywise_from_dof_geometry_P607_P664(mode, n):
    """M_eps built entry by entry from the DoF-level definitions, on random masks where I1, I2,
    I3 and I_V all differ, compared EXACTLY with the oracle:
      M_ii(p,p) = (eps_ii - 1) I_i[p] + 1;
      Trivial:  M_ij(p,p) = eps_ij I_V[p], M_ji = conj;
      CrossDoF: M_ij(p,q) = eps_ij (I_i[p] + I_j[q]) / 8 for the four E^j DoFs q nearest to the
                E^i DoF p (|dx_i| = |dx_j| = h/2 on the two axes of i, j, same coordinate on the
                third: the interpolation of P:640-654), M_ji(q,p) = conj(eps_ij)(I_i[p]+I_j[q])/8
                (S_ij = (I_i T_ij + T_ij I_j)/2)."""
    rng = np.random.default_rng(100 + n)
    masks = (rng.random((4, n, n, n)) < 0.5).astype(np.uint8)
    assert all((masks[a] != masks[b]).any() for a in range(4) for b in range(a))
    e = synth.eps_sdd() if mode != "diagonal" else np.diag([0.3, 0.55, 0.8]).astype(complex)
    N3 = n ** 3
    I = [masks[c].reshape(-1).astype(float) for c in range(4)]
    ref = np.zeros((3 * N3, 3 * N3), complex)
    for i in range(3):
        for p in range(N3):
            ref[i * N3 + p, i * N3 + p] = (e[i, i].real - 1.0) * I[i][p] + 1.0
    pos = _dof_positions(n)
    for i, j in [(0, 1), (0, 2), (1, 2)]:
        if mode == "trivial":
            for p in range(N3):
                ref[i * N3 + p, j * N3 + p] = e[i, j] * I[3][p]
                ref[j * N3 + p, i * N3 + p] = np.conj(e[i, j]) * I[3][p]
        elif mode == "crossdof":
            third = 3 - i - j
            for p in range(N3):
                d = pos[j] - pos[i][p]
                d = d - n * np.round(d / n)            # periodic minimum image
                near = (np.abs(np.abs(d[:, i]) - 0.5) < 1e-12) & (np.abs(np.abs(d[:, j]) - 0.5) < 1e-12) \
                    & (np.abs(d[:, third]) < 1e-12)
                qs = np.nonzero(near)[0]
                assert qs.size == 4
                for q in qs:
                    w = (I[i][p] + I[j][q]) / 8.0
                    ref[i * N3 + p, j * N3 + q] = e[i, j] * w
                    ref[j * N3 + q, i * N3 + p] = np.conj(e[i, j]) * w
    M = O.permittivity_matrix(e, masks, mode).toarray()
    assert np.array_equal(M, ref)


def test_permittivity_special_cases():
    n = 4
    A = np.eye(3)
    e = synth.eps_pseudochiral()
    M = O.permittivity_matrix(e, synth.make_masks("vacuum", A, n), "crossdof")
    assert abs(M - np.eye(3 * n ** 3)).max() == 0          # VACUUM -> identity
    one = np.ones(3 * n ** 3)
    Mt = O.permittivity_matrix(e, synth.make_masks("full", A, n), "trivial")
    ref = np.concatenate([np.full(n ** 3, e[r].sum()) for r in range(3)])
    assert np.allclose(Mt @ one, ref, atol=1e-15)
    d = np.diag([0.2, 0.5, 0.9]).astype(complex)
    masks = synth.make_masks("random", A, n, seed=1)
    assert abs(O.permittivity_matrix(d, masks, "diagonal") - O.permittivity_matrix(d, masks, "crossdof")).max() == 0


def test_hpd_report_spec_examples():
    r = O.hpd_report(np.diag([0.5, 0.5, 0.5]))
    assert r == {"assumption1": True, "sdd": True, "zero_offdiag": True, "guaranteed": True}
    r = O.hpd_report(synth.eps_pseudochiral())
    assert r["assumption1"] and r["zero_offdiag"] and r["guaranteed"]
    r = O.hpd_report(np.diag([1.5, 0.5, 0.5]))
    assert not r["assumption1"] and not r["guaranteed"]


# ---------------------------------------------------------------- Fourier apply, preconditioner
@pytest.mark.parametrize("lat", ["sc", "fcc"])
def test_fourier_apply_is_conjugated_operator_P523(lat):
    n = 4
    A = synth.lattice(lat)
    F = O.dft_matrix(n)
    F3 = np.kron(np.kron(F, F), F)
    Z = np.zeros_like(F3)
    F3b = np.block([[F3, Z, Z], [Z, F3, Z], [Z, Z, F3]])
    op = O.PenalizedOperator(n, np.array([0.9, 2.0, -1.3]), A, synth.eps_sdd(), synth.make_masks("random", A, n, seed=2))
    x = synth.random_block(n, 2, seed=4)
    ref = (F3b.conj().T @ op.dense() @ F3b @ x.T).T
    assert np.allclose(op.apply_fourier(x), ref, atol=1e-9)


@pytest.mark.parametrize("lat,k", [("sc", (0.5, 0.2, -0.1)), ("fcc", (PI, PI, PI)), ("sc", (0, 0, 0))])
def test_preconditioner_inverts_vacuum_operator_P532(lat, k):
    """With M = I the Fourier-space operator IS K_P, so K_P^{-1} Op x = x
    ("preconditioned vacuum = identity"); at k = 0 mode 0 passes through (R7)."""
    n = 5
    A = synth.lattice(lat)
    k = np.array(k)
    op = O.PenalizedOperator(n, k, A, np.eye(3), synth.make_masks("vacuum", A, n))
    x = synth.random_block(n, 2, seed=11)
    if not np.any(k):
        x[:, [0, n ** 3, 2 * n ** 3]] = 0.0
    y = op.apply_fourier(x)
    assert np.allclose(O.precond_fourier(n, k, A, op.gamma, y), x, atol=1e-10)


@pytest.mark.parametrize("lat,k", [("sc", (0.5, 0.2, -0.1)), ("fcc", (PI, PI, PI))])
def test_eps_preconditioner_is_kp_in_vacuum(lat, k):
    """With M = I the eps-weighted preconditioner (reading R16) reduces to the paper's K_P^{-1}
    (P:530-548): (I - Pi)/|kappa|^2 + Pi/(gamma |kappa|^2)."""
    n = 5
    A = synth.lattice(lat)
    k = np.array(k)
    masks = synth.make_masks("vacuum", A, n)
    g = O.gamma_rule(k)
    r = synth.random_block(n, 2, seed=12)
    ref = O.precond_fourier(n, k, A, g, r)
    got = O.precond_eps_fourier(n, k, A, g, synth.eps_pseudochiral(), masks, "crossdof", r)
    assert np.allclose(got, ref, rtol=0, atol=1e-12 * np.abs(ref).max())


@pytest.mark.parametrize("lat,c", [("sc", 13.0), ("fcc", 0.2)])
def test_eps_preconditioner_inverts_homogeneous_operator(lat, c):
    """For a homogeneous isotropic medium (every mask 1, eps_1 = c I, so M = c I) the eps-weighted
    preconditioner is the exact inverse of the Fourier-space operator: T Op x = x (k != 0, no zero
    modes).  The check goes through the oracle's sparse operator, not the symbols."""
    n = 4
    A = synth.lattice(lat)
    k = np.array([0.7, -1.1, 0.4])
    masks = synth.make_masks("full", A, n)
    op = O.PenalizedOperator(n, k, A, c * np.eye(3), masks, "crossdof")
    x = synth.random_block(n, 2, seed=13)
    y = op.apply_fourier(x)
    got = O.precond_eps_fourier(n, k, A, op.gamma, c * np.eye(3), masks, "crossdof", y)
    assert np.allclose(got, x, rtol=0, atol=1e-9 * np.abs(x).max())


def test_eps_preconditioner_hermitian_positive():
    """T is Hermitian positive definite on an inhomogeneous pseudochiral medium (k != 0):
    <x, T y> = <T x, y>, <x, T x> > 0."""
    n = 6
    A = synth.lattice("fcc")
    k = np.array([PI, PI, PI])
    masks = synth.make_masks("fcc_diamond", A, n)
    e = synth.eps_pseudochiral()
    g = O.gamma_rule(k)
    x, y = synth.random_block(n, 2, seed=14)
    Tx, Ty = O.precond_eps_fourier(n, k, A, g, e, masks, "crossdof", np.stack([x, y]))
    assert abs(np.vdot(x, Ty) - np.vdot(Tx, y)) <= 1e-12 * abs(np.vdot(x, Ty))
    assert np.vdot(x, Tx).real > 0 and abs(np.vdot(x, Tx).imag) <= 1e-12 * np.vdot(x, Tx).real


def test_kappa_symbols_match_operator():
    """kappa_i(m) are the eigenvalues of Dhat_i on the Fourier basis."""
    n = 4
    A = synth.lattice("fcc")
    k = np.array([0.3, 1.9, -2.2])
    D = O.shifted_blocks(n, k, A)
    kap = O.kappa_symbols(n, k, A).reshape(3, -1)
    x = synth.random_block(n, 1, seed=6)[0][: n ** 3]
    H = np.fft.ifftn(x.reshape(n, n, n), norm="ortho").ravel()
    for i in range(3):
        y = np.fft.fftn((D[i] @ H).reshape(n, n, n), norm="ortho").ravel()
        assert np.allclose(y, kap[i] * x, atol=1e-11)


# ---------------------------------------------------------------- iterative vs dense
@pytest.mark.parametrize("lat,k", [("sc", (PI, PI, PI)), ("fcc", (0.7, -1.1, 2.0)), ("sc", (0, 0, 0))])
def test_iterative_matches_dense(lat, k):
    n = 6
    A = synth.lattice(lat)
    masks = synth.make_masks("random", A, n, seed=21)
    op = O.PenalizedOperator(n, np.array(k), A, synth.eps_pseudochiral(), masks)
    wd = O.eigs_dense(op, 8)
    wi, res = O.eigs_iterative(op, 8, tol=1e-9, seed=1)
    assert np.allclose(wi, wd, rtol=1e-8)
