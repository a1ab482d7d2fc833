"""GPU eigenvalue parity: pc_bands (device LOBPCG) against the oracle's eigenvalues and closed forms.
Bar: relative error <= 1e-8 (BASELINE.json north_star)."""
import math
import os

import numpy as np
import pytest

import synth
from oracle import pc_oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
PI = math.pi
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
TOL = 1e-7   # Res_j tolerance for parity runs (reading R13): eigenvalue error ~ Res^2 / gap


@pytest.fixture(scope="module")
def api():
    from paper_2511_17107_b200 import api as a
    return a


def golden(name):
    rows = {}
    for line in open(os.path.join(GOLD, name)):
        if line.startswith("#") or not line.strip():
            continue
        key, *vals = line.split()
        rows[key] = np.array([float(v) for v in vals])
    return rows


def rel(a, b):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b)) / np.abs(np.asarray(b))))


def test_c1_vacuum_n8_golden(api):
    """BASELINE config 1: SC vacuum n=8, 6 smallest vs closed form, from the default
    (plane-wave) start and from a seeded Gaussian start, both at the parity tolerance 1e-7."""
    g = golden("c1_vacuum_n8.txt")
    ctx = api.pc_create(np.eye(3), 8, np.eye(3), np.zeros((4, 8, 8, 8), np.uint8))
    kp = [[PI, PI, PI], [PI / 7, 3 * PI / 5, 4 * PI / 13]]
    r = api.pc_bands(ctx, kp, nev=6, tol=TOL)
    assert (r["status"] == 0).all()
    assert rel(r["omega2"][0], g["k_a"]) <= 1e-8
    assert rel(r["omega2"][1], g["k_b"]) <= 1e-8
    api.pc_set_option(ctx, "start", 0)
    for seed in (0, 7):
        r = api.pc_bands(ctx, kp, nev=6, tol=TOL, seed=seed)
        assert (r["status"] == 0).all()
        assert rel(r["omega2"], np.stack([g["k_a"], g["k_b"]])) <= 1e-8


def test_c1_vacuum_iterations(api):
    """In vacuum K_P^{-1} is the exact inverse (M_eps = I), so the preconditioned Rayleigh
    quotient is constant (Prop. P:550-569; "converges in <= 2 iterations").  Reading R17
    (DESIGN.md): that holds for a start block inside the invariant subspace -- the transverse plane
    waves, which are the vacuum eigenvectors, converge at once -- while from a
    generic start T = A^{-1} makes LOBPCG an inverse iteration with Rayleigh-Ritz: the residual of band j
    falls by at least lambda_j / lambda_{b+1} per step, which bounds the iteration count."""
    g = golden("c1_vacuum_n8.txt")
    ctx = api.pc_create(np.eye(3), 8, np.eye(3), np.zeros((4, 8, 8, 8), np.uint8))
    kb = [PI / 7, 3 * PI / 5, 4 * PI / 13]
    api.pc_set_option(ctx, "start_noise", 0.0)
    r = api.pc_bands(ctx, [kb], nev=6, tol=TOL)
    assert r["iters"].max() <= 2 and rel(r["omega2"][0], g["k_b"]) <= 1e-8
    api.pc_set_option(ctx, "start", 0)
    b = 6 + 6
    lam = _vacuum_closed(8, np.array(kb), np.eye(3), b + 1, O.gamma_rule(kb))
    rate = lam[5] / lam[b]
    res0 = 1e5  # >= ||A|| x relative admixture of a unit Gaussian start at n = 8 (gamma max|kappa|^2 ~ 3e4)
    bound = int(np.ceil(np.log(TOL / res0) / np.log(rate))) + 2
    r = api.pc_bands(ctx, [kb], nev=6, tol=TOL, seed=3)
    assert r["status"][0] == 0 and rel(r["omega2"][0], g["k_b"]) <= 1e-8
    assert r["iters"][0] <= bound, (r["iters"][0], bound, rate)


def test_homogeneous_n8_golden(api):
    g = golden("homog_n8_R.txt")
    for lat in ("sc", "fcc"):
        A = synth.lattice(lat)
        ctx = api.pc_create(A, 8, synth.eps_pseudochiral(), synth.make_masks("full", A, 8))
        r = api.pc_bands(ctx, [[PI, PI, PI]], nev=10, tol=TOL)
        assert r["status"][0] == 0
        assert rel(r["omega2"][0], g[lat]) <= 1e-8


@pytest.mark.parametrize("lat,n,k,eps,geo", [
    ("sc", 6, (PI, PI, PI), "pc", "random"),
    ("fcc", 6, (0.7, -1.1, 2.0), "pc", "random"),
    ("sc", 8, (0.0, 0.0, 0.0), "pc", "random"),
    ("fcc", 8, (PI, PI, PI), "sdd", "random"),
    ("bcc", 6, (PI, 0, PI), "sdd", "random"),
    ("sc", 8, (0.2, 0.1, 0.0), "iso", "sphere"),
])
@pytest.mark.parametrize("tmap", [0, 1])
def test_bands_match_dense_oracle(api, lat, n, k, eps, geo, tmap):
    """Both block-update kernels (cp.async tiles / TMA tensor copies; n = 6 has a ragged last tile)."""
    A = synth.lattice(lat)
    e = {"pc": synth.eps_pseudochiral(), "sdd": synth.eps_sdd(), "iso": synth.eps_isotropic(13.0)}[eps]
    masks = synth.make_masks(geo, A, n, seed=31)
    ctx = api.pc_create(A, n, e, masks)
    api.pc_set_option(ctx, "update_tmap", tmap)
    r = api.pc_bands(ctx, [k], nev=10, tol=TOL)
    assert r["status"][0] == 0
    op = O.PenalizedOperator(n, np.array(k), A, e, masks)
    ref = O.eigs_dense(op, 10)
    assert rel(r["omega2"][0], ref) <= 1e-8
    assert (r["resid"][0] <= TOL).all()


def test_bands_match_iterative_oracle_fcc_n16(api):
    """Pseudochiral FCC diamond (the bench's workload shape) at n=16 vs the oracle's SciPy solve."""
    A = synth.lattice("fcc")
    n = 16
    e = synth.eps_pseudochiral()
    masks = synth.make_masks("fcc_diamond", A, n)
    k = np.array([PI, PI, PI])
    ctx = api.pc_create(A, n, e, masks)
    r = api.pc_bands(ctx, [k], nev=10, tol=TOL)
    assert r["status"][0] == 0
    op = O.PenalizedOperator(n, k, A, e, masks)
    ref, res = O.eigs_iterative(op, 10, tol=1e-10, seed=3)
    assert rel(r["omega2"][0], ref) <= 1e-8


def _vacuum_closed(n, k, A, nev, gamma):
    h = 1.0 / n
    th = 2 * PI * np.arange(n) / n
    l1 = (1 - np.exp(-1j * th)) / h
    l0 = (1 + np.exp(-1j * th)) / 2
    B = np.linalg.inv(A)
    g1 = [l1[None, None, :], l1[None, :, None], l1[:, None, None]]
    g0 = [l0[None, None, :], l0[None, :, None], l0[:, None, None]]
    k2 = 0
    for i in range(3):
        k2 = k2 + np.abs(sum(B[j, i] * g1[j] for j in range(3)) + 1j * k[i] * g0[i]) ** 2
    k2 = np.broadcast_to(k2, (n, n, n)).ravel()
    vals = np.sort(np.concatenate([k2, k2, gamma * k2]))
    if not np.any(k):
        vals = vals[3:]
    return vals[:nev]


@pytest.mark.parametrize("lat,n,k", [("sc", 64, (0.5, 0.0, 0.0)), ("fcc", 128, (PI, PI, PI)), ("sc", 32, (0, 0, 0))])
def test_bands_vacuum_closed_form_large(api, lat, n, k):
    """Vacuum at the large sizes: {|kappa|^2 (x2), gamma |kappa|^2}, including
    the spurious gamma-modes inside the window (reading R11)."""
    A = synth.lattice(lat)
    ctx = api.pc_create(A, n, np.eye(3), np.zeros((4, n, n, n), np.uint8))
    r = api.pc_bands(ctx, [k], nev=10, tol=1e-6)
    ref = _vacuum_closed(n, np.array(k), A, 10, O.gamma_rule(k))
    assert rel(r["omega2"][0], ref) <= 1e-8


def test_bands_homogeneous_closed_form_n32(api):
    """Homogeneous pseudochiral FCC at n=32: per-mode 3x3 closed form."""
    n, A, e = 32, synth.lattice("fcc"), synth.eps_pseudochiral()
    k = np.array([PI / 2, 2 * PI, PI / 2])
    h = 1.0 / n
    th = 2 * PI * np.arange(n) / n
    l1 = (1 - np.exp(-1j * th)) / h
    l0 = (1 + np.exp(-1j * th)) / 2
    B = np.linalg.inv(A)
    m1, m2, m3 = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    m = [m1.ravel(), m2.ravel(), m3.ravel()]
    kap = np.stack([sum(B[j, i] * l1[m[j]] for j in range(3)) + 1j * k[i] * l0[m[i]] for i in range(3)], axis=1)
    KA = np.zeros((kap.shape[0], 3, 3), complex)
    KA[:, 0, 1], KA[:, 0, 2], KA[:, 1, 0] = -kap[:, 2], kap[:, 1], kap[:, 2]
    KA[:, 1, 2], KA[:, 2, 0], KA[:, 2, 1] = -kap[:, 0], -kap[:, 1], kap[:, 0]
    t12 = l0[m[0]] * np.conj(l0[m[1]])
    Mh = np.broadcast_to(e, (kap.shape[0], 3, 3)).copy()
    Mh[:, 0, 1] = e[0, 1] * t12
    Mh[:, 1, 0] = np.conj(e[0, 1]) * np.conj(t12)
    gamma = O.gamma_rule(k)
    K = KA @ Mh @ np.conj(np.transpose(KA, (0, 2, 1))) + gamma * np.conj(kap)[:, :, None] * kap[:, None, :]
    ref = np.sort(np.linalg.eigvalsh(K).ravel())[:10]
    ctx = api.pc_create(A, n, e, synth.make_masks("full", A, n))
    r = api.pc_bands(ctx, [k], nev=10, tol=TOL)
    assert rel(r["omega2"][0], ref) <= 1e-8


def test_bands_determinism_and_sharding_seed(api):
    """Same seed -> bit-identical; results of k-point i do not depend on how the path is split."""
    A = synth.lattice("sc")
    n = 8
    masks = synth.make_masks("random", A, n, seed=2)
    ctx = api.pc_create(A, n, synth.eps_pseudochiral(), masks)
    ks = synth.kpath("sc", 2)[:4]
    r1 = api.pc_bands(ctx, ks, nev=6, tol=1e-8, seed=5)
    r2 = api.pc_bands(ctx, ks, nev=6, tol=1e-8, seed=5)
    assert np.array_equal(r1["omega2"], r2["omega2"]) and np.array_equal(r1["iters"], r2["iters"])
    api.pc_set_option(ctx, "kindex_offset", 2)
    r3 = api.pc_bands(ctx, ks[2:], nev=6, tol=1e-8, seed=5)
    assert np.array_equal(r3["omega2"], r1["omega2"][2:])


def test_bands_eigenvectors(api):
    n, A = 8, synth.lattice("fcc")
    e = synth.eps_pseudochiral()
    masks = synth.make_masks("random", A, n, seed=12)
    ctx = api.pc_create(A, n, e, masks)
    k = np.array([0.4, 1.0, -0.3])
    ev = torch.empty(6, 3 * n ** 3, dtype=torch.complex128, device="cuda")
    r = api.pc_bands(ctx, [k], nev=6, tol=1e-9, evecs=ev)
    V = ev.cpu().numpy()
    op = O.PenalizedOperator(n, k, A, e, masks)
    AV = op.apply_fourier(V)
    res = np.linalg.norm(AV - r["omega2"][0][:, None] * V, axis=1)
    assert np.allclose(np.linalg.norm(V, axis=1), 1.0, atol=1e-12)
    assert res.max() <= 1e-8


def test_bands_warm_start_path_continuation(api):
    """Warm start: same eigenvalues as cold starts (both to TOL, compared at 1e-8
    relative against the dense oracle at n=8), path includes Gamma (cold there), and fewer total
    iterations than the cold path."""
    from paper_2511_17107_b200 import bands
    A = synth.lattice("fcc")
    n = 8
    e = synth.eps_pseudochiral()
    masks = synth.make_masks("random", A, n, seed=21)
    kp = synth.kpath("fcc", 4)[6:16]  # U -> L -> Gamma -> ... (contains k = 0)
    ctx = api.pc_create(A, n, e, masks)
    cold = bands.solve_local(ctx, kp, list(range(len(kp))), 6, TOL, 500, 0)
    warm = bands.solve_warm([ctx], kp, list(range(len(kp))), 6, TOL, 500, 0)
    assert (cold[3] == 0).all() and (warm[3] == 0).all()
    for i, k in enumerate(kp):
        op = O.PenalizedOperator(n, k, A, e, masks)
        ref = O.eigs_dense(op, 6)
        assert rel(warm[0][i], ref) <= 1e-8
        assert rel(cold[0][i], ref) <= 1e-8
    assert warm[2].sum() < cold[2].sum()


@pytest.mark.parametrize("opts", [{"fuse_resid": 0}, {"gram_refresh": 1}, {"trim_locked": 0}, {"sticky_lock": 1},
                                  {"update_tmap": 0}, {"w_guard": -1}, {"w_guard": 2},
                                  {"precond": 1}, {"precond": 1, "trim_locked": 0},
                                  {"precond": 1, "precond_fuse": 0}, {"precond": 1, "fuse_xex": 0},
                                  {"guard": 1}, {"guard": 2}, {"guard": 3}, {"guard": 4}, {"guard": 5}, {"guard": 7},
                                  {"guard": 8}, {"guard": 3, "precond": 1}, {"guard": 7, "update_tmap": 0}])
def test_bands_option_variants(api, opts):
    """Alternative LOBPCG paths (unfused residual, cp.async update tiles, full Gram every iteration, W for
    guard columns, other block widths, the eps-weighted preconditioner) reach the dense oracle's eigenvalues."""
    A = synth.lattice("fcc")
    n = 8
    e = synth.eps_pseudochiral()
    masks = synth.make_masks("fcc_diamond", A, n)
    k = np.array([PI / 7, 3 * PI / 5, 4 * PI / 13])
    ctx = api.pc_create(A, n, e, masks)
    for key, v in opts.items():
        api.pc_set_option(ctx, key, v)
    r = api.pc_bands(ctx, [k], nev=10, tol=TOL)
    assert r["status"][0] == 0
    op = O.PenalizedOperator(n, k, A, e, masks)
    assert rel(r["omega2"][0], O.eigs_dense(op, 10)) <= 1e-8


@pytest.mark.parametrize("guard", [4, 5, 6])
def test_bands_nev20_block_sizes(api, guard):
    """C5's band count (nev = 20, b = nev + guard = 24-26, the library maximum) at n = 8 against the dense oracle: every
    block width maps onto the TMA update stage layout (the X block ends on a DMMA k-step)."""
    A = synth.lattice("fcc")
    n = 8
    e = synth.eps_pseudochiral()
    masks = synth.make_masks("fcc_diamond", A, n)
    k = np.array([PI, PI, PI])
    ctx = api.pc_create(A, n, e, masks)
    api.pc_set_option(ctx, "guard", guard)
    r = api.pc_bands(ctx, [k], nev=20, tol=TOL)
    assert r["status"][0] == 0
    op = O.PenalizedOperator(n, k, A, e, masks)
    assert rel(r["omega2"][0], O.eigs_dense(op, 20)) <= 1e-8


@pytest.mark.parametrize("nev", [1, 2, 3, 5, 7, 12, 16])
@pytest.mark.parametrize("precond", [0, 1])
def test_bands_nev_sweep(api, nev, precond):
    """Band counts 1-16 (block widths 7-22 with the default guard) with both preconditioners against
    the dense oracle (FCC diamond, pseudochiral, n = 8, a generic k)."""
    A = synth.lattice("fcc")
    n = 8
    e = synth.eps_pseudochiral()
    masks = synth.make_masks("fcc_diamond", A, n)
    k = np.array([0.3, -1.1, 2.0])
    ctx = api.pc_create(A, n, e, masks)
    api.pc_set_option(ctx, "precond", precond)
    r = api.pc_bands(ctx, [k], nev=nev, tol=TOL)
    assert r["status"][0] == 0
    op = O.PenalizedOperator(n, k, A, e, masks)
    assert rel(r["omega2"][0], O.eigs_dense(op, nev)) <= 1e-8


def test_bands_full_size_c4_properties(api):
    """The bench workload itself (C4: FCC diamond, pseudochiral, n = 128, 10 bands, tol 1e-5, one path
    k-point), with both preconditioners: sampled eigenpairs checked through the ORACLE's sparse operator
    (too large for its eigensolver): residual ||Op v - w v|| <= 1.5 tol, Rayleigh quotient = w, V^H V = I,
    and the two preconditioners agree on every eigenvalue."""
    W = synth.WORKLOADS["C4"]
    A, e, n = W.A(), W.eps1(), W.n
    masks = W.masks()
    k = W.kpoints()[7]
    om = {}
    for pre in (0, 1):
        ctx = api.pc_create(A, n, e, masks)
        api.pc_set_option(ctx, "precond", pre)
        ev = torch.empty(10, 3 * n ** 3, dtype=torch.complex128, device="cuda")
        r = api.pc_bands(ctx, [k], nev=10, tol=1e-5, evecs=ev)
        assert r["status"][0] == 0
        om[pre] = r["omega2"][0]
        if pre == 1:
            V = ev.cpu().numpy()
            G = V.conj() @ V.T
            assert np.abs(G - np.eye(10)).max() <= 1e-10
            op = O.PenalizedOperator(n, k, A, e, masks)
            for j in (0, 4, 9):
                Av = op.apply_fourier(V[j][None, :])[0]
                assert np.linalg.norm(Av - om[1][j] * V[j]) <= 1.5e-5
                assert abs(np.vdot(V[j], Av).real - om[1][j]) <= 1e-9 * om[1][j]
        ctx.close()
    assert rel(om[0], om[1]) <= 1e-9


# ------------------------------------------------------- config-size eigenvalue parity (C2, C3, C4)
def _golden_sets():
    """tests/golden/c{2,3,4}_*.txt, written by tests/golden/gen_goldens.py from the oracle only."""
    out = []
    for name in ("c2_sc_sphere_n32.txt", "c3_sc_sc_curv_n64.txt", "c4_fcc_fcc_diamond_n128.txt"):
        path = os.path.join(GOLD, name)
        if os.path.exists(path):
            g = golden(name)
            for key in g:
                if key.startswith("ev"):
                    out.append(pytest.param(name, int(key[2:]), id=f"{name[:2]}-k{key[2:]}"))
    return out


@pytest.mark.parametrize("name,ki", _golden_sets())
def test_bands_match_oracle_goldens_config_size(api, name, ki):
    """North-star target (BASELINE.json): all 10 bands at the benchmark configurations against the
    oracle's eigenvalues (SciPy LOBPCG on the oracle's sparse operator, tol <= 2e-8), relative <= 1e-8.
    C2: SC sphere n = 32, the whole 33-point path; C3: SC-CURV pseudochiral n = 64; C4: FCC diamond
    pseudochiral n = 128 (the bench workload) at X, a generic U-L point and L.  PAPER.md:1055-1064,
    1080-1095."""
    wname = {"c2": "C2", "c3": "C3", "c4": "C4"}[name[:2]]
    W = synth.WORKLOADS[wname]
    g = golden(name)
    k = g[f"k{ki}"]
    assert np.allclose(k, W.kpoints()[ki], rtol=0, atol=1e-15)
    ref = g[f"ev{ki}"]
    ctx = _ctx_cache(wname)
    api.pc_set_option(ctx, "kindex_offset", ki)
    r = api.pc_bands(ctx, [k], nev=W.nev, tol=TOL, maxit=1000)
    assert r["status"][0] == 0
    assert rel(r["omega2"][0], ref) <= 1e-8, (r["omega2"][0], ref)


_CTX = {}


def _ctx_cache(wname):
    from paper_2511_17107_b200 import api as a
    if wname not in _CTX:
        _CTX.clear()  # one workload context alive at a time (C4 needs ~17 GB of workspace)
        W = synth.WORKLOADS[wname]
        _CTX[wname] = a.pc_create(W.A(), W.n, W.eps1(), W.masks())
    return _CTX[wname]



@pytest.mark.parametrize("wname,kb,idx", [("C2", 4, list(range(0, 8))), ("C3", 3, [4, 5, 6])])
def test_bands_kbatch_equals_single(api, wname, kb, idx):
    """k-points solved in lock step (option kbatch: one multi-k apply, two host
    synchronisations per iteration for the whole batch) give the eigenvalues, residuals and iteration
    counts of one-at-a-time solves (same arithmetic per k), and match the oracle goldens where they exist."""
    W = synth.WORKLOADS[wname]
    name = {"C2": "c2_sc_sphere_n32.txt", "C3": "c3_sc_sc_curv_n64.txt"}[wname]
    g = golden(name)
    kp = W.kpoints()[idx]
    ctx = api.pc_create(W.A(), W.n, W.eps1(), W.masks())
    ref = np.zeros((len(idx), W.nev))
    its = np.zeros(len(idx), dtype=int)
    for t, ki in enumerate(idx):
        api.pc_set_option(ctx, "kindex_offset", ki)
        r = api.pc_bands(ctx, kp[t:t + 1], nev=W.nev, tol=TOL)
        ref[t], its[t] = r["omega2"][0], r["iters"][0]
    api.pc_set_option(ctx, "kbatch", kb)
    api.pc_set_option(ctx, "kindex_offset", idx[0])  # consecutive indices: start blocks keyed as above
    r = api.pc_bands(ctx, kp, nev=W.nev, tol=TOL)
    assert (r["status"] == 0).all()
    assert np.array_equal(r["iters"], its)
    assert rel(r["omega2"], ref) <= 1e-12
    for t, ki in enumerate(idx):
        if f"ev{ki}" in g:
            assert rel(r["omega2"][t], g[f"ev{ki}"]) <= 1e-8


def test_bands_kbatch_eigenvectors(api):
    """Lock-step batch with eigenvector output (k-major, one block per k-point): every
    returned pair is an eigenpair of the oracle operator of its own k, including k = 0."""
    n, A = 8, synth.lattice("fcc")
    e = synth.eps_pseudochiral()
    masks = synth.make_masks("random", A, n, seed=12)
    ctx = api.pc_create(A, n, e, masks)
    kp = np.array([[0.4, 1.0, -0.3], [0.0, 0.0, 0.0], [PI, PI, PI]])
    api.pc_set_option(ctx, "kbatch", 3)
    ev = torch.empty(3 * 6, 3 * n ** 3, dtype=torch.complex128, device="cuda")
    r = api.pc_bands(ctx, kp, nev=6, tol=1e-9, evecs=ev)
    assert (r["status"] == 0).all()
    V = ev.cpu().numpy()
    for i, k in enumerate(kp):
        op = O.PenalizedOperator(n, k, A, e, masks)
        Vi = V[6 * i:6 * (i + 1)]
        res = np.linalg.norm(op.apply_fourier(Vi) - r["omega2"][i][:, None] * Vi, axis=1)
        assert np.allclose(np.linalg.norm(Vi, axis=1), 1.0, atol=1e-12)
        assert res.max() <= 1e-8
        assert rel(r["omega2"][i], O.eigs_dense(op, 6)) <= 1e-8
