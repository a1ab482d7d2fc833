"""Input generator checks (SPEC lattice/geometry examples)."""
import math

import numpy as np

import synth

PI = math.pi


def test_lattices_P965():
    for kind in ("sc", "fcc", "bcc"):
        A = synth.lattice(kind)
        assert np.allclose(A @ np.linalg.inv(A), np.eye(3), atol=1e-14)
    assert np.array_equal(synth.lattice("fcc")[:, 0], [0, 0.5, 0.5])
    assert np.array_equal(synth.lattice("bcc")[:, 0], [-0.5, 0.5, 0.5])


def test_kpath_counts():
    assert synth.kpath("sc", 8).shape == (33, 3)
    assert synth.kpath("fcc", 8).shape == (49, 3)
    assert synth.kpath("fcc", 32).shape == (193, 3)
    p = synth.kpath("sc", 2, ["G", "X"])
    assert np.allclose(p, [[0, 0, 0], [PI / 2, 0, 0], [PI, 0, 0]])
    assert np.allclose(synth.kpath("sc", 4, ["G", "R"])[-1], [PI, PI, PI])


def test_eps_pseudochiral_eigs_S289():
    ev = np.linalg.eigvalsh(synth.eps_pseudochiral(13, 0.875))
    assert np.allclose(ev, [0.034905248199, 0.076923076923, 0.169520632815], atol=1e-12)
    e = synth.eps_extreme()
    assert np.allclose(np.linalg.eigvalsh(e), [1e-5, 1e-3, 1e-1], rtol=1e-9)


def test_masks_basic():
    A = np.eye(3)
    assert synth.make_masks("vacuum", A, 4).sum() == 0
    assert synth.make_masks("full", A, 4).min() == 1
    m = synth.make_masks("sphere", A, 16)
    vol = 4 / 3 * PI * 0.345 ** 3
    assert abs(m[3].mean() - vol) < 0.02
    c = synth.contains("sc_curv", np.array([[0.5, 0.5, 0.5]]), A)
    assert c[0]
    g = synth.contains("bcc_sg", np.array([[0.0, 0, 0], [0.125, 0, 0]]), A)
    assert not g.any()
    # determinism
    assert np.array_equal(synth.make_masks("fcc_diamond", synth.lattice("fcc"), 8),
                          synth.make_masks("fcc_diamond", synth.lattice("fcc"), 8))


def test_random_block_layout():
    x = synth.random_block(4, 3, seed=1)
    assert x.shape == (3, 192) and x.flags.c_contiguous and x.dtype == np.complex128
    s = synth.random_block(8, 1, seed=2, kind="smooth").reshape(3, 8, 8, 8)
    assert s[:, 4, 4, 4].sum() == 0 and np.abs(s[:, 1, 1, 1]).sum() > 0
