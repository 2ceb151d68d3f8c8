"""Pins of the fp64 oracle against what the paper and mathematics fix
(never against the oracle itself).  CPU only.  See DESIGN.md "Oracle pins".
"""
import json
import math
import os

import mpmath as mp
import numpy as np
import pytest
from scipy import integrate, optimize

import oracle
from oracle import qform, recon
from workloads import make_config
from workloads.configs import seeded_rng

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


def paper_to_config(v):
    """paper frame (x beam, y fan, z out of fan) -> config frame (x out of fan, y fan, z beam)."""
    return [v[2], v[1], v[0]]


# ---------------------------------------------------------------- factors --
@pytest.mark.parametrize("ex", GOLD["G_so"])
def test_G_so_worked(ex):
    assert oracle.G_so(paper_to_config(ex["r_paper"])) == pytest.approx(ex["value"], rel=ex["rtol"])


@pytest.mark.parametrize("ex", GOLD["G_od"])
def test_G_od_worked(ex):
    assert oracle.G_od(paper_to_config(ex["s_paper"])) == pytest.approx(ex["value"], rel=ex["rtol"])


@pytest.mark.parametrize("ex", GOLD["theta"])
def test_theta_worked(ex):
    th = oracle.theta(paper_to_config(ex["r_paper"]), paper_to_config(ex["rp_paper"]))
    assert th == pytest.approx(ex["value"], rel=ex["rtol"])


@pytest.mark.parametrize("ex", GOLD["bragg_energy"])
def test_bragg_worked(ex):
    assert qform.bragg_energy(ex["q"], ex["theta"]) == pytest.approx(ex["value"], rel=ex["rtol"])


@pytest.mark.parametrize("ex", GOLD["spectral_factor_flat"])
def test_spectral_factor_worked(ex):
    assert qform.spectral_factor(ex["theta"], ex["q"], lambda E: 1.0) == pytest.approx(ex["value"], rel=ex["rtol"])


def test_dtheta_small_angle_and_zero_pitch():
    # on-axis far pixel dtheta ~ pitch/|s|; pitch 0 -> 0
    r = [0.0, 0.0, 400.0]
    rp = [0.0, 0.0, 1400.0]
    assert oracle.dtheta(r, rp, 0.0) == 0.0
    assert oracle.dtheta(r, rp, 1.0) == pytest.approx(2 * math.atan(0.5 / 1000.0), rel=1e-14)
    rp2 = [30.0, 20.0, 1400.0]
    s = np.subtract(rp2, r)
    assert oracle.dtheta(r, rp2, 0.4) == pytest.approx(0.4 * math.hypot(s[1], s[2]) / np.dot(s, s), rel=1e-6)


def test_dtheta_mpmath():
    """dtheta = angle between the two edge-midpoint vectors via 40-digit acos."""
    mp.mp.dps = 40
    rng = np.random.default_rng(5)
    for _ in range(20):
        r = [0.0, rng.uniform(-50, 50), rng.uniform(300, 600)]
        rp = [rng.uniform(10, 150), rng.uniform(-60, 60), 1000.0]
        p = rng.uniform(0.1, 2.0)
        a = mp.matrix([rp[0] + p / 2 - r[0], rp[1] - r[1], rp[2] - r[2]])
        b = mp.matrix([rp[0] - p / 2 - r[0], rp[1] - r[1], rp[2] - r[2]])
        ref = mp.acos((a.T * b)[0] / (mp.norm(a) * mp.norm(b)))
        assert oracle.dtheta(r, rp, p) == pytest.approx(float(ref), rel=1e-12)


# ---------------------------------------------------- single-voxel geometry --
def single_voxel_cfg(ne=8, nq=101, q_min=0.0, q_max=1.0, e_lo=30.0, e_hi=120.0, phi=None,
                     energy=None, open_mask=True, det=(4, 4), det_pitch=1.5):
    cfg = make_config(0)
    d = cfg.desc()
    d.update(ny=1, nz=1, y_min=-1.5, y_max=2.5, z_min=440.0, z_max=446.0, nq=nq, q_min=q_min,
             q_max=q_max, ne=ne, det_nx=det[0], det_ny=det[1], det_pitch=det_pitch)
    if energy is None:
        width = (e_hi - e_lo) / ne
        energy = e_lo + (np.arange(ne) + 0.5) * width
    if phi is None:
        phi = np.linspace(1.0, 0.3, ne)
    d["energy_kev"], d["phi"] = np.asarray(energy, float), np.asarray(phi, float)
    d["mask"] = np.ones_like(d["mask"]) if open_mask else d["mask"]
    return d


def mp_pair(d, y_r, z_r, x_d, y_d):
    """P, sin(theta/2) from 40-digit mpmath, acos forms (independent of the C code)."""
    mp.mp.dps = 40
    r = mp.matrix([0, y_r, z_r])
    rp = mp.matrix([x_d, y_d, d["det_z"]])
    s = rp - r
    gso = mp.mpf(z_r) / (mp.mpf(y_r) ** 2 + mp.mpf(z_r) ** 2) ** mp.mpf(1.5)
    god = s[2] / mp.norm(s) ** 3
    th = mp.acos((r.T * s)[0] / (mp.norm(r) * mp.norm(s)))
    h = mp.mpf(d["det_pitch"]) / 2
    a = s + mp.matrix([h, 0, 0])
    b = s - mp.matrix([h, 0, 0])
    dth = mp.acos((a.T * b)[0] / (mp.norm(a) * mp.norm(b)))
    P = d["scale"] * gso * god * dth * (1 + mp.cos(th) ** 2) * mp.cos(th / 2)
    return P, mp.sin(th / 2)


def centres(d):
    G = oracle.Geometry(d)
    yv, zv = G.voxel_centres()
    xd, yd = G.det_centres()
    return G, yv[0], zv[0], xd, yd


def test_single_voxel_constant_profile():
    """(i) f = 1 on all nodes, all u_k inside [0, Q-1] => g = P sum_k phi_k E_k."""
    d = single_voxel_cfg()
    G, yr, zr, xd, yd = centres(d)
    g = G.forward(np.ones(G.f_shape))
    S = float(np.sum(d["phi"] * d["energy_kev"]))
    for ix in range(d["det_nx"]):
        for jy in range(d["det_ny"]):
            P, _ = mp_pair(d, yr, zr, xd[ix], yd[jy])
            assert g[ix, jy] == pytest.approx(float(P) * S, rel=1e-12)


def test_single_voxel_linear_profile():
    """(ii) f_j = q_j is reproduced exactly by linear interpolation
    => g = P (sin(theta/2)/hc) sum_k phi_k E_k^2  (Bragg)."""
    d = single_voxel_cfg()
    G, yr, zr, xd, yd = centres(d)
    q = d["q_min"] + np.arange(d["nq"]) * ((d["q_max"] - d["q_min"]) / (d["nq"] - 1))
    g = G.forward(np.broadcast_to(q, G.f_shape))
    S2 = np.sum(d["phi"] * d["energy_kev"] ** 2)
    for ix in range(d["det_nx"]):
        for jy in range(d["det_ny"]):
            P, sh = mp_pair(d, yr, zr, xd[ix], yd[jy])
            ref = P * sh / mp.mpf("12.3984193") * mp.mpf(S2)
            assert g[ix, jy] == pytest.approx(float(ref), rel=1e-11)


def test_single_voxel_one_energy_one_node():
    """(iii) K = 1, f one-hot at node j0 => g = P phi E Lambda(u - j0),
    u = (E sin(theta/2)/hc - q_0)/dq."""
    d = single_voxel_cfg(ne=1, energy=[60.0], phi=[0.7], nq=41, q_min=0.0, q_max=0.4)
    G, yr, zr, xd, yd = centres(d)
    dq = mp.mpf(0.4) / 40
    for j0 in range(8, 30):
        f = np.zeros(G.f_shape)
        f[0, 0, j0] = 1.0
        g = G.forward(f)
        for ix in range(d["det_nx"]):
            for jy in range(d["det_ny"]):
                P, sh = mp_pair(d, yr, zr, xd[ix], yd[jy])
                u = (60 * sh / mp.mpf("12.3984193")) / dq
                lam = max(mp.mpf(0), 1 - abs(u - j0))
                assert g[ix, jy] == pytest.approx(float(P * mp.mpf(0.7) * 60 * lam), rel=1e-10, abs=1e-30)


def test_single_voxel_backward_moments():
    """w one-hot at a pixel: sum_j b_j = P sum phi E and sum_j q_j b_j = P (sh/hc) sum phi E^2
    (partition of unity and linear reproduction of the hat basis)."""
    d = single_voxel_cfg()
    G, yr, zr, xd, yd = centres(d)
    q = d["q_min"] + np.arange(d["nq"]) * ((d["q_max"] - d["q_min"]) / (d["nq"] - 1))
    for ix, jy in [(0, 0), (1, 3), (3, 2)]:
        w = np.zeros(G.g_shape)
        w[ix, jy] = 2.5
        b = G.backward(w)[0, 0]
        P, sh = mp_pair(d, yr, zr, xd[ix], yd[jy])
        S1 = np.sum(d["phi"] * d["energy_kev"])
        S2 = np.sum(d["phi"] * d["energy_kev"] ** 2)
        assert b.sum() == pytest.approx(float(2.5 * P * S1), rel=1e-12)
        assert (q * b).sum() == pytest.approx(float(2.5 * P * sh / mp.mpf("12.3984193") * S2), rel=1e-11)


def test_energy_form_matches_paper_q_form():
    """Continuum pin of reading R2: sum_k phi_k E_k f~(u_k) (1+cos^2) cos(theta/2)
    -> hc^2 int S(theta,q) f(q) dq as the grids refine."""
    e_lo, e_hi, e_max = 20.0, 150.0, 155.0
    K = 3000
    width = (e_hi - e_lo) / K
    E = e_lo + (np.arange(K) + 0.5) * width

    def Phi(e):
        return (e_max - e) / e if e_lo <= e <= e_hi else 0.0

    phi = np.array([Phi(e) for e in E]) * width
    d = single_voxel_cfg(ne=K, energy=E, phi=phi, nq=4001, q_min=0.0, q_max=0.8, det=(3, 1))
    d.update(det_cx=60.0, det_pitch=40.0, det_cy=0.0, mask_pitch=10.0)  # pixels at x = 20, 60, 100 mm
    G, yr, zr, xd, yd = centres(d)
    q = d["q_min"] + np.arange(d["nq"]) * (0.8 / 4000)

    def fq(x):
        return math.exp(-((x - 0.2) ** 2) / (2 * 0.03 ** 2)) + 0.5 * math.exp(-((x - 0.33) ** 2) / (2 * 0.02 ** 2))

    g = G.forward(np.array([fq(x) for x in q]).reshape(G.f_shape))
    for ix in range(3):
        fac = G.pair(0, 0, ix, 0)
        th = fac["theta"]
        sh = math.sin(th / 2)
        lo, hi = e_lo * sh / qform.HC, e_hi * sh / qform.HC
        integral, _ = integrate.quad(lambda x: qform.spectral_factor(th, x, Phi) * fq(x), lo, hi,
                                     limit=400, epsabs=0, epsrel=1e-12)
        ref = fac["G_so"] * fac["G_od"] * fac["dtheta"] * qform.HC ** 2 * integral
        assert g[ix, 0] == pytest.approx(ref, rel=2e-5)


# ------------------------------------------------------- operator properties --
def test_dense_matrix_matches_loops_config0():
    cfg = make_config(0)
    G = oracle.Geometry(cfg)
    A = oracle.dense_A(cfg)
    rng = seeded_rng(0, 3)
    f = rng.random(G.f_shape)
    w = rng.random(G.g_shape)
    g = G.forward(f)
    b = G.backward(w)
    assert np.abs(A @ f.ravel() - g.ravel()).max() <= 1e-13 * np.abs(g).max()
    assert np.abs(A.T @ w.ravel() - b.ravel()).max() <= 1e-13 * np.abs(b).max()


def test_dense_matrix_matches_loops_energy_resolving():
    cfg = make_config(0, energy_resolving=1)
    G = oracle.Geometry(cfg)
    A = oracle.dense_A(cfg)
    assert A.shape == (16 * 16 * 8, 64 * 16)
    rng = seeded_rng(0, 4)
    f = rng.random(G.f_shape)
    w = rng.random(G.g_shape)
    g = G.forward(f)
    b = G.backward(w)
    assert np.abs(A @ f.ravel() - g.ravel()).max() <= 1e-13 * np.abs(g).max()
    assert np.abs(A.T @ w.ravel() - b.ravel()).max() <= 1e-13 * np.abs(b).max()


def test_energy_resolved_sums_to_integrating():
    """Reading R12: sum_k g[r', k] equals the energy-integrating g."""
    cfg = make_config(0)
    g = oracle.Geometry(cfg).forward(cfg.f)
    ge = oracle.Geometry(cfg, energy_resolving=1).forward(cfg.f)
    np.testing.assert_allclose(ge.sum(-1), g, rtol=1e-13, atol=1e-13 * g.max())


@pytest.mark.parametrize("ci,npairs", [(0, 20), (1, 1)])
def test_adjoint_identity(ci, npairs):
    """<A x, y> = <x, A^T y> to 1e-10 (north_star)."""
    cfg = make_config(ci)
    G = oracle.Geometry(cfg)
    rng = seeded_rng(ci, 5)
    for _ in range(npairs):
        x = rng.random(G.f_shape)
        y = rng.random(G.g_shape)
        lhs = np.vdot(G.forward(x), y)
        rhs = np.vdot(x, G.backward(y))
        assert abs(lhs - rhs) <= 1e-10 * abs(lhs)


def test_adjoint_identity_energy_resolving():
    cfg = make_config(0, energy_resolving=1)
    G = oracle.Geometry(cfg)
    rng = seeded_rng(0, 6)
    for _ in range(5):
        x = rng.random(G.f_shape)
        y = rng.random(G.g_shape)
        assert abs(np.vdot(G.forward(x), y) - np.vdot(x, G.backward(y))) <= 1e-10 * abs(np.vdot(G.forward(x), y))


def test_nonnegativity_and_linearity():
    cfg = make_config(0)
    G = oracle.Geometry(cfg)
    rng = seeded_rng(0, 7)
    f, h = rng.random(G.f_shape), rng.random(G.f_shape)
    gf, gh = G.forward(f), G.forward(h)
    assert (gf >= 0).all() and (G.backward(rng.random(G.g_shape)) >= 0).all()
    np.testing.assert_allclose(G.forward(2.5 * f + 0.75 * h), 2.5 * gf + 0.75 * gh, rtol=1e-13,
                               atol=1e-14 * gf.max())


# ----------------------------------------------------------------- the mask --
def test_mask_all_open_and_all_closed():
    cfg = make_config(0)
    d = cfg.desc()
    d_open = dict(d, mask=np.ones_like(d["mask"]))
    d_closed = dict(d, mask=np.zeros_like(d["mask"]))
    Go, Gc = oracle.Geometry(d_open), oracle.Geometry(d_closed)
    # every config-0 ray crosses inside the raster (SURVEY.md §8(d) coverage), so T == 1
    for iy in range(8):
        for iz in range(8):
            for ix in range(0, 16, 3):
                for jy in range(0, 16, 3):
                    assert Go.pair(iy, iz, ix, jy)["T"] == 1.0
    f = cfg.f.astype(np.float64)
    assert (Gc.forward(f) == 0).all()
    assert (Gc.backward(np.ones(Gc.g_shape)) == 0).all()


def test_mask_single_hole_vs_exact_rays():
    """Single open cell: T = 1 exactly for the pairs whose ray crosses z = z_m
    inside that cell, decided in exact rational arithmetic (fractions) from the
    fp64 centre coordinates; only rays within 1e-9 cells of an edge may differ."""
    from fractions import Fraction as Fr
    cfg = make_config(0)
    d = cfg.desc()
    hole = (18, 17)
    m = np.zeros_like(d["mask"])
    m[hole] = 1
    d = dict(d, mask=m)
    G = oracle.Geometry(d)
    yv, zv = G.voxel_centres()
    xd, yd = G.det_centres()
    mp_ = Fr(d["mask_pitch"])
    m0x = Fr(d["mask_cx"]) - Fr(d["mask_nx"]) * mp_ / 2
    m0y = Fr(d["mask_cy"]) - Fr(d["mask_ny"]) * mp_ / 2
    n_hit = 0
    for iy in range(8):
        for iz in range(8):
            for ix in range(16):
                for jy in range(16):
                    yr, zr, x, y = Fr(yv[iy]), Fr(zv[iz]), Fr(xd[ix]), Fr(yd[jy])
                    t = (Fr(d["mask_z"]) - zr) / (Fr(d["det_z"]) - zr)
                    ux = (t * x - m0x) / mp_
                    uy = (yr + t * (y - yr) - m0y) / mp_
                    exact = (math.floor(ux), math.floor(uy)) == hole
                    near = min(abs(ux - round(ux)), abs(uy - round(uy))) < Fr(1, 10 ** 9)
                    T = G.pair(iy, iz, ix, jy)["T"]
                    if not near:
                        assert T == (1.0 if exact else 0.0)
                    n_hit += int(T)
    assert n_hit > 0


# ------------------------------------------------------- Lemma 1 and update --
@pytest.mark.parametrize("ex", GOLD["lemma1"])
def test_lemma_worked(ex):
    assert recon.lemma_minimizer(ex["a"], ex["b"], ex["c"]) == pytest.approx(ex["value"], abs=1e-15)


def test_lemma_unbounded_case():
    assert recon.lemma_minimizer(0.0, -1.0, 2.0) == np.inf


def test_lemma_vs_bounded_search():
    """1000 random draws vs a bracketing numerical minimiser of the Lemma's f(x)."""
    rng = np.random.default_rng(11)
    for _ in range(1000):
        a = rng.uniform(0, 3) if rng.random() > 0.2 else 0.0
        b = rng.uniform(-3, 3)
        if a == 0.0:
            b = abs(b) + 0.1
        c = rng.uniform(0, 3) if rng.random() > 0.1 else 0.0
        x = recon.lemma_minimizer(a, b, c)

        def fun(v):
            return 0.5 * a * v * v + b * v - (c * math.log(v) if c > 0 else 0.0)
        hi = max(10.0, 4 * x)
        res = optimize.minimize_scalar(fun, bounds=(1e-12, hi), method="bounded",
                                       options={"xatol": 1e-12})
        assert fun(x) <= fun(res.x) + 1e-9
        assert x == pytest.approx(res.x, rel=1e-5, abs=1e-6)


def test_lemma_root_vs_mpmath_textbook():
    mp.mp.dps = 50
    rng = np.random.default_rng(12)
    for _ in range(200):
        a, b, c = rng.uniform(1e-6, 1e-2), rng.uniform(1.0, 1e4), rng.uniform(0, 1e3)
        ref = (-mp.mpf(b) + mp.sqrt(mp.mpf(b) ** 2 + 4 * mp.mpf(a) * mp.mpf(c))) / (2 * mp.mpf(a))
        assert recon.lemma_minimizer(a, b, c) == pytest.approx(float(ref), rel=1e-14)


def test_update_minimises_separable_surrogate():
    """Eq. f_update equals the numerical argmin of the per-voxel separable
    surrogate  -f^_j b2_j ln x + b1_j x + beta sum_{k in N_j} psi(2x - f^_j - f^_k)
    (PAPER.md:673, 681-697 with quadratic psi, symmetric N)."""
    rng = np.random.default_rng(13)
    ny, nz, nq = 5, 4, 3
    f_hat = rng.uniform(0.1, 2, (ny, nz, nq))
    b1 = rng.uniform(0.5, 3, (ny, nz, nq))
    b2 = rng.uniform(0.1, 3, (ny, nz, nq))
    for beta in (0.0, 0.01, 0.7):
        out = recon.update(f_hat, b1, b2, beta)
        for (i, j, q) in [(0, 0, 0), (2, 1, 1), (4, 3, 2), (2, 0, 1)]:
            nb = [f_hat[i + di, j + dj, q] for di, dj in ((1, 0), (-1, 0), (0, 1), (0, -1))
                  if 0 <= i + di < ny and 0 <= j + dj < nz]

            def sur(x):
                return (-f_hat[i, j, q] * b2[i, j, q] * math.log(x) + b1[i, j, q] * x
                        + beta * sum(0.5 * (2 * x - f_hat[i, j, q] - fk) ** 2 for fk in nb))
            res = optimize.minimize_scalar(sur, bounds=(1e-9, 50), method="bounded", options={"xatol": 1e-12})
            assert out[i, j, q] == pytest.approx(res.x, rel=1e-6)


def test_update_beta0_is_mlem():
    rng = np.random.default_rng(14)
    f_hat, b1, b2 = rng.uniform(0.1, 2, (3, 3, 4)), rng.uniform(0.5, 3, (3, 3, 4)), rng.uniform(0, 3, (3, 3, 4))
    np.testing.assert_allclose(recon.update(f_hat, b1, b2, 0.0), f_hat * b2 / b1, rtol=1e-15)


def test_penalty_double_counts_pairs():
    f = np.zeros((2, 1, 1))
    f[0, 0, 0] = 1.0
    # one unordered neighbour pair, counted once from each side: 2 * psi(1) = 1
    assert recon.penalty(f) == pytest.approx(1.0)


# --------------------------------------------------------------- EM (Alg 5) --
def _em_setup(beta_data=True):
    cfg = make_config(0)
    G = oracle.Geometry(cfg)
    f_true = cfg.f.astype(np.float64)
    l = G.forward(f_true)
    s = 50.0 / l.mean()
    G = oracle.Geometry(cfg, scale=s)
    rng = seeded_rng(0, 8)
    y = rng.poisson(G.forward(f_true) + 1.0).astype(np.float64)
    r = np.ones(G.g_shape)
    b1 = G.backward(np.ones(G.g_shape))
    return G, f_true, y, r, b1


def test_em_monotone_unpenalised():
    """beta = 0: L is non-increasing (north_star; EM surrogate majorisation)."""
    G, f_true, y, r, b1 = _em_setup()
    f0 = np.full(G.f_shape, max((y - r).sum(), 1.0) / b1.sum())
    trace = []
    recon.em_iterate(G, f0, y, r, b1, 0.0, 15, trace)
    assert all(b <= a * (1 + 1e-12) for a, b in zip(trace, trace[1:]))
    assert trace[-1] < trace[0]


def test_em_monotone_penalised():
    G, f_true, y, r, b1 = _em_setup()
    f0 = np.full(G.f_shape, max((y - r).sum(), 1.0) / b1.sum())
    trace = []
    recon.em_iterate(G, f0, y, r, b1, 5e-3, 15, trace)
    assert all(b <= a * (1 + 1e-12) for a, b in zip(trace, trace[1:]))


def test_em_fixed_point():
    """y = A f*, r = 0, beta = 0 => f* is a fixed point where b1 > 0."""
    cfg = make_config(0)
    G = oracle.Geometry(cfg)
    f_star = np.full(G.f_shape, 0.3)
    y = G.forward(f_star)
    b1 = G.backward(np.ones(G.g_shape))
    f1 = recon.em_iterate(G, f_star, y, np.zeros(G.g_shape), b1, 0.0, 1)[0]
    seen = b1 > 0
    np.testing.assert_allclose(f1[seen], f_star[seen], rtol=1e-12)


def test_effective_terms_config0():
    """every config-0 energy is in range for every pair (fraction 1.00)."""
    cfg = make_config(0)
    pairs, open_, terms = oracle.Geometry(cfg).count_terms()
    assert pairs == 64 * 256 and terms == open_ * 8


# ---- round-2 pins: centres, objective, ratio guard, term counting, adjoint ----
@pytest.mark.parametrize("ci,iy,iz,yz", [
    # config 0 (BASELINE configs[0]): y in [-8, 8], z in [400, 416], 8 x 8 pixels of 2 mm
    (0, 0, 0, (-7.0, 401.0)), (0, 7, 7, (7.0, 415.0)), (0, 3, 5, (-1.0, 411.0)),
    # config 1: y in [-40, 40] (64 x 1.25 mm), z in [350, 550] (64 x 3.125 mm)
    (1, 0, 0, (-39.375, 351.5625)), (1, 63, 63, (39.375, 548.4375)), (1, 32, 0, (0.625, 351.5625)),
])
def test_voxel_centres_hand_values(ci, iy, iz, yz):
    """Reading R9 (pixel centres at min + (i + 1/2) pitch), pinned by hand values
    of the configs' stated extents -- for oracle.c and the numpy restatement."""
    G = oracle.Geometry(make_config(ci))
    assert G.voxel_centre(iy, iz) == pytest.approx(yz, abs=1e-12)
    yv, zv = G.voxel_centres()
    assert (yv[iy], zv[iz]) == pytest.approx(yz, abs=1e-12)


@pytest.mark.parametrize("ci,ix,jy,xy", [
    # config 0: 16 x 16 pixels of 1.5 mm centred at x = +24 (near edge at x = 12 + 0.75), y = 0
    (0, 0, 0, (12.75, -11.25)), (0, 15, 15, (35.25, 11.25)), (0, 8, 7, (24.75, -0.75)),
    # config 1: 128 x 128 pixels of 0.8 mm, near x edge at 12 mm
    (1, 0, 0, (12.4, -50.8)), (1, 127, 127, (114.0, 50.8)),
])
def test_detector_centres_hand_values(ci, ix, jy, xy):
    G = oracle.Geometry(make_config(ci))
    assert G.det_centre(ix, jy) == pytest.approx(xy, abs=1e-12)
    xd, yd = G.det_centres()
    assert (xd[ix], yd[jy]) == pytest.approx(xy, abs=1e-12)


def test_neg_loglik_hand_values():
    """L = sum_i (l_i + r_i) - y_i ln(l_i + r_i) (reading R15:
    the constant sum ln y_i! dropped) at points computed by hand."""
    assert recon.neg_loglik([1.0], [1.0], [0.0]) == pytest.approx(1.0, abs=1e-15)        # 1 - 1 ln 1
    e = np.e
    assert recon.neg_loglik([e - 1.0], [2.0], [1.0]) == pytest.approx(e - 2.0, rel=1e-15)  # z = e: e - 2
    assert recon.neg_loglik([0.0], [0.0], [0.0]) == 0.0                                 # 0 ln 0 := 0
    assert recon.neg_loglik([3.0], [0.0], [2.0]) == pytest.approx(5.0, rel=1e-15)         # y = 0: L = z
    # r enters z: l = 1, r = 3, y = 4 -> 4 - 4 ln 4
    assert recon.neg_loglik([1.0], [4.0], [3.0]) == pytest.approx(4.0 - 4.0 * np.log(4.0), rel=1e-14)
    # a sum over pixels
    assert recon.neg_loglik([1.0, 1.0, 0.5], [1.0, 0.0, 1.0], [0.0, 1.0, 0.5]) == pytest.approx(
        1.0 + 2.0 + 1.0, rel=1e-15)
    # J = L + beta R: two voxels (y neighbours) 1 and 3 in one q node -> R = psi(-2) + psi(2) = 4
    f = np.array([1.0, 3.0]).reshape(2, 1, 1)
    assert recon.penalty(f) == pytest.approx(4.0)
    assert recon.objective([1.0], [1.0], [0.0], f, 0.25) == pytest.approx(1.0 + 0.25 * 4.0)


def test_ratio_guard_branches():
    """Reading R14: y / (l + r); 0 where y = z = 0; y / 1e-12 where z = 0 < y."""
    out = recon.ratio([0.0, 0.0, 1.0, 2.0], [0.0, 5.0, 2.0, 0.0], [0.0, 0.0, 1.0, 0.0])
    assert out[0] == 0.0
    assert out[1] == pytest.approx(5e12, rel=1e-15)
    assert out[2] == pytest.approx(1.0, rel=1e-15)
    assert out[3] == 0.0


@pytest.mark.parametrize("over", [dict(q_min=0.15, q_max=0.25, nq=9), dict(q_min=0.06, q_max=0.12, nq=5),
                                  dict(q_min=0.0, q_max=0.9, nq=40)])
def test_count_terms_out_of_range_energies(over):
    """oracle_count_terms' in-range predicate (-1 < u_k < Q) against a count from
    the dense matrix's own pair angles (oracle/dense.py: half-angle atan2, a
    different formula) on geometries whose q grid cuts off part of the Bragg
    reach (so some energies fall outside) and one that contains all of it."""
    cfg = make_config(0)
    d = cfg.desc()
    d.update(over)
    pairs, open_, terms = oracle.Geometry(d).count_terms()
    pa = oracle.dense.pair_arrays(d)
    E = np.asarray(d["energy_kev"], float)
    dq = (d["q_max"] - d["q_min"]) / (d["nq"] - 1)
    u = (E[None, None, :] * np.sin(0.5 * pa["theta"])[..., None] / oracle.HC - d["q_min"]) / dq
    inr = (u > -1.0) & (u < d["nq"]) & (pa["T"][..., None] == 1.0)
    assert pairs == pa["T"].size
    assert open_ == int((pa["T"] == 1.0).sum())
    assert terms == int(inr.sum())
    if over["q_max"] < 0.5:
        assert terms < open_ * d["ne"]  # the predicate actually cuts


def test_adjoint_identity_config1_20_pairs():
    """<A x, y> = <x, A^T y> to 1e-10 for 20 random pairs on config 1:
    4 with the full operators and 16 with y supported on a random 1/16 of the
    pixels (the pixel-restricted loops oracle_forward_pixels / oracle_backward_pixels
    of Alg. 6, so the CPU suite stays within minutes).  Signed y: no positivity to
    hide a sign error."""
    cfg = make_config(1)
    G = oracle.Geometry(cfg)
    rng = seeded_rng(1, 6)
    npx = cfg.n_det
    for i in range(20):
        x = rng.random(G.f_shape)
        y = rng.random(G.g_shape) - 0.5
        if i < 4:
            ax = G.forward(x)
            lhs, rhs = np.vdot(ax, y), np.vdot(x, G.backward(y))
        else:
            pix = np.sort(rng.choice(npx, npx // 16, replace=False))
            ax = G.forward_pixels(x, pix)
            lhs = np.vdot(ax, y.ravel()[pix])
            ys = np.zeros(npx)
            ys[pix] = y.ravel()[pix]
            rhs = np.vdot(x, G.backward_pixels(ys.reshape(G.g_shape), pix))
        assert abs(lhs - rhs) <= 1e-10 * np.linalg.norm(ax) * np.linalg.norm(y), i
