"""Pins of the oracle's reconstruction extensions (SURVEY.md §8(f) rows f2 and
f4): the Huber edge-preserving potential in the update, and ordered subsets
(Alg. 6) with the symmetry-preserving partition of Fig. 6.  CPU only; every
check is against the paper's text, a worked example or a mathematical
property -- never the oracle against itself.
"""
import json
import math
import os

import numpy as np
import pytest
from scipy import optimize

import oracle
from oracle import recon
from workloads import make_config
from workloads.configs import seeded_rng

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


# ------------------------------------------------------------------ Huber --
@pytest.mark.parametrize("ex", GOLD["huber"])
@pytest.mark.parametrize("delta", [0.1, 1.0, 3.0])
def test_huber_worked(ex, delta):
    pen = recon.Penalty("huber", delta)
    x = ex["x_over_delta"] * delta
    assert float(pen.psi(x)) == pytest.approx(ex["psi_over_delta2"] * delta ** 2, abs=1e-15)
    assert float(pen.psi_dot(x)) == pytest.approx(ex["psi_dot_over_delta"] * delta, abs=1e-15)
    assert float(pen.omega(x)) == pytest.approx(ex["omega"], abs=1e-15)


def test_huber_properties():
    """Symmetric, C1 at |x| = delta, psi_dot = d psi / dx (finite differences),
    omega = psi_dot / x, and the large-delta limit is the quadratic potential."""
    d = 0.7
    pen = recon.Penalty("huber", d)
    x = np.linspace(-5, 5, 2001)
    np.testing.assert_array_equal(pen.psi(x), pen.psi(-x))
    h = 1e-6
    away = np.abs(np.abs(x) - d) > 2 * h  # central differences are O(h) only at the kink
    np.testing.assert_allclose(((pen.psi(x + h) - pen.psi(x - h)) / (2 * h))[away], pen.psi_dot(x)[away], atol=1e-8)
    nz = np.abs(x) > 1e-9
    np.testing.assert_allclose(pen.omega(x)[nz], pen.psi_dot(x)[nz] / x[nz], rtol=1e-14)
    assert float(pen.psi(d * (1 + 1e-12))) == pytest.approx(0.5 * d * d, rel=1e-9)
    big = recon.Penalty("huber", 1e9)
    np.testing.assert_allclose(big.psi(x), 0.5 * x * x, rtol=1e-15)


def test_huber_curvature_majorises():
    """The quadratic surrogate with curvature omega(x^) = psi_dot(x^)/x^
    majorises psi_delta and touches it at x^ (Huber's
    condition) -- the property the monotone descent of Alg. 5 rests on."""
    pen = recon.Penalty("huber", 0.5)
    xs = np.linspace(-4, 4, 801)
    for xh in (-3.0, -0.5, -0.2, 0.0, 0.3, 0.5, 2.0):
        sur = pen.psi(xh) + pen.psi_dot(xh) * (xs - xh) + 0.5 * pen.omega(xh) * (xs - xh) ** 2
        assert (sur >= pen.psi(xs) - 1e-14).all()
        assert float(pen.psi(xh)) == pytest.approx(float(pen.psi(xh) + 0 * xh))


def test_huber_penalty_constant_image_and_pair():
    pen = recon.Penalty("huber", 0.25)
    assert recon.penalty(np.full((3, 4, 2), 1.7), pen) == 0.0
    f = np.zeros((2, 1, 1))
    f[0, 0, 0] = 1.0
    # one unordered neighbour pair, counted twice: 2 psi(1) = 2 (0.25 - 0.03125)
    assert recon.penalty(f, pen) == pytest.approx(2 * (0.25 * 1.0 - 0.5 * 0.25 ** 2))


def test_huber_update_minimises_separable_surrogate():
    """Eq. f_update with omega / psi_dot of the Huber potential equals the
    numerical argmin of the voxel's separable surrogate
      -f^_j b2_j ln x + b1_j x + beta sum_{k in N_j} psi^_{x^}(2x - f^_j - f^_k),
    psi^ the quadratic surrogate expanded at x^ = f^_j - f^_k
    (PAPER.md:673, 681-698)."""
    rng = np.random.default_rng(21)
    ny, nz, nq = 5, 4, 3
    f_hat = rng.uniform(0.1, 2, (ny, nz, nq))
    b1 = rng.uniform(0.5, 3, (ny, nz, nq))
    b2 = rng.uniform(0.1, 3, (ny, nz, nq))
    for delta in (0.05, 0.4, 5.0):
        pen = recon.Penalty("huber", delta)
        for beta in (0.01, 0.7, 3.0):
            out = recon.update(f_hat, b1, b2, beta, pen)
            for (i, j, q) in [(0, 0, 0), (2, 1, 1), (4, 3, 2), (2, 0, 1), (1, 2, 0)]:
                nb = [f_hat[i + di, j + dj, q] for di, dj in ((1, 0), (-1, 0), (0, 1), (0, -1))
                      if 0 <= i + di < ny and 0 <= j + dj < nz]
                fj = f_hat[i, j, q]

                def psihat(x, xh):
                    return float(pen.psi(xh) + pen.psi_dot(xh) * (x - xh) + 0.5 * pen.omega(xh) * (x - xh) ** 2)

                def sur(x):
                    return (-fj * b2[i, j, q] * math.log(x) + b1[i, j, q] * x
                            + beta * sum(psihat(2 * x - fj - fk, fj - fk) for fk in nb))
                res = optimize.minimize_scalar(sur, bounds=(1e-9, 50), method="bounded", options={"xatol": 1e-12})
                assert out[i, j, q] == pytest.approx(res.x, rel=1e-6)


def _em_setup():
    cfg = make_config(0)
    G = oracle.Geometry(cfg)
    f_true = cfg.f.astype(np.float64)
    s = 50.0 / G.forward(f_true).mean()
    G = oracle.Geometry(cfg, scale=s)
    y = seeded_rng(0, 8).poisson(G.forward(f_true) + 1.0).astype(np.float64)
    r = np.ones(G.g_shape)
    b1 = G.backward(np.ones(G.g_shape))
    f0 = np.full(G.f_shape, max((y - r).sum(), 1.0) / b1.sum())
    return G, f_true, y, r, b1, f0


def test_em_monotone_huber():
    """beta > 0 with the Huber potential: J is non-increasing (surrogate
    majorisation)."""
    G, f_true, y, r, b1, f0 = _em_setup()
    trace = []
    recon.em_iterate(G, f0, y, r, b1, 2e-2, 12, trace, recon.Penalty("huber", 0.05))
    assert all(b <= a * (1 + 1e-12) for a, b in zip(trace, trace[1:]))
    assert trace[-1] < trace[0]


# ------------------------------------------------------ subsets (Alg. 6) --
def test_partition_fig6_groups():
    """The paper's own example (Fig. 6)."""
    ex = GOLD["partition_fig6"]
    sub = recon.symmetric_partition(ex["M"], ex["N"], ex["rho_z"], ex["rho_y"])
    assert sub.max() + 1 == ex["P"]
    for row in range(ex["M"]):
        ids = {sub[row, j - 1] for grp in ex["same_subset_columns_1based"] for j in grp}
        assert len(ids) == 1
    for col in range(ex["N"]):
        ids = {sub[i - 1, col] for grp in ex["same_subset_rows_1based"] for i in grp}
        assert len(ids) == 1
    # column 2 is NOT in column 1's subset (different n)
    assert sub[0, 1] != sub[0, 0]


@pytest.mark.parametrize("M,N,rz,ry", [(32, 64, 8, 16), (16, 16, 4, 8), (8, 12, 2, 6), (128, 128, 8, 16),
                                       (4, 4, 1, 2), (6, 10, 3, 2)])
def test_partition_closure_and_balance(M, N, rz, ry):
    """Every subset is closed under the up-down mirror (row i <-> M-1-i), the
    left-right mirror (col j <-> N-1-j) and +-rho_y column translation
    (PAPER.md:381-387); P = rho_z rho_y / 2 equal subsets of M N / P pixels."""
    sub = recon.symmetric_partition(M, N, rz, ry)
    P = rz * ry // 2
    assert sub.max() + 1 == P and sub.min() == 0
    np.testing.assert_array_equal(np.bincount(sub.ravel()), np.full(P, M * N // P))
    np.testing.assert_array_equal(sub, sub[::-1, :])
    np.testing.assert_array_equal(sub, sub[:, ::-1])
    np.testing.assert_array_equal(sub[:, ry:], sub[:, :-ry])


def test_partition_rejects_bad_steps():
    for args in [(32, 64, 3, 16), (32, 64, 8, 15), (32, 60, 8, 16), (31, 64, 8, 16)]:
        with pytest.raises(ValueError):
            recon.symmetric_partition(*args)


def test_subset_completeness():
    """sum_p A_p f = A f and sum_p A_p^T w = A^T w (SPEC.md:621 AC10): the
    subsets partition the measurement space."""
    cfg = make_config(0)
    G = oracle.Geometry(cfg)
    sub = recon.symmetric_partition(cfg.det_nx, cfg.det_ny, 4, 8)
    f = cfg.f.astype(np.float64)
    w = seeded_rng(5, 1).uniform(0, 1, G.g_shape)
    g = G.forward(f)
    parts = [np.where(sub == p, g, 0.0) for p in range(16)]
    np.testing.assert_array_equal(sum(parts), g)
    back = sum(G.backward(w * (sub == p)) for p in range(16))
    np.testing.assert_allclose(back, G.backward(w), rtol=1e-13, atol=0)


def test_osem_one_subset_is_em():
    """P = 1 (rho_z = 1, rho_y = 2): Alg. 6 reduces to Alg. 5."""
    G, f_true, y, r, b1, f0 = _em_setup()
    sub = recon.symmetric_partition(16, 16, 1, 2)
    assert sub.max() == 0
    a = recon.osem_iterate(G, f0, y, r, sub, 1e-2, 3)
    b = recon.em_iterate(G, f0, y, r, b1, 1e-2, 3)
    for x, z in zip(a, b):
        np.testing.assert_allclose(x, z, rtol=1e-13)


def test_osem_accelerates():
    """16 symmetry-preserving subsets: the objective after ONE outer iteration
    is below EM's after 8 iterations (SPEC.md:617 AC7, the desk-scale analogue
    of the paper's ~76x with 64 subsets)."""
    G, f_true, y, r, b1, f0 = _em_setup()
    sub = recon.symmetric_partition(16, 16, 4, 8)
    beta = 1e-3
    t_os, t_em = [], []
    recon.osem_iterate(G, f0, y, r, sub, beta, 1, t_os)
    recon.em_iterate(G, f0, y, r, b1, beta, 8, t_em)
    assert t_os[-1] <= t_em[-1]


def test_restricted_operators_equal_masked_definitions():
    """forward_pixels / backward_pixels (sums over the subset's pixels only)
    equal the masked full operators (A f)|_p and A^T (w 1_p) -- the oracle's
    two ways of writing A_p agree."""
    cfg = make_config(0)
    G = oracle.Geometry(cfg)
    sub = recon.symmetric_partition(cfg.det_nx, cfg.det_ny, 4, 8).ravel()
    f = cfg.f.astype(np.float64)
    w = seeded_rng(6, 1).uniform(0, 1, G.g_shape)
    g = G.forward(f).ravel()
    for p in (0, 5, 15):
        pix = np.flatnonzero(sub == p)
        np.testing.assert_allclose(G.forward_pixels(f, pix), g[pix], rtol=1e-15)
        np.testing.assert_allclose(G.backward_pixels(w, pix), G.backward(w * (sub == p).reshape(G.g_shape)),
                                   rtol=1e-12, atol=1e-300)


def test_osem_restricted_matches_definition():
    G, f_true, y, r, b1, f0 = _em_setup()
    sub = recon.symmetric_partition(16, 16, 4, 8)
    a = recon.osem_iterate(G, f0, y, r, sub, 1e-3, 1)
    b = recon.osem_iterate(G, f0, y, r, sub, 1e-3, 1, restricted=True)
    np.testing.assert_allclose(a[0], b[0], rtol=1e-10)
