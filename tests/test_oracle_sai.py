"""Pins of the oracle's scatter-angle interpolation (SAI, PAPER.md:220-233;
SURVEY.md §8(f) row f3): the spectral-angular factor of each pair evaluated
at the nearest of N uniformly spaced angles (reading R22).  CPU only.
"""
import math

import mpmath as mp
import numpy as np
import pytest

import oracle
from workloads import make_config
from workloads.configs import seeded_rng

TH_MIN, TH_MAX = 0.2 * math.pi / 180.0, math.pi / 6.0  # reading R22 ("0.2 to pi/6")


def sai(cfg, n, **kw):
    return oracle.Geometry(cfg, sai_n_theta=n, sai_theta_min=TH_MIN, sai_theta_max=TH_MAX, **kw)


def test_nearest_angle_rule():
    O = sai(make_config(0), 251)
    h = (TH_MAX - TH_MIN) / 250
    for i in (0, 1, 17, 125, 250):
        t = TH_MIN + i * h
        assert O.sai_angle(t) == pytest.approx(t, abs=1e-15)
        assert O.sai_angle(t + 0.49 * h) == pytest.approx(t, abs=1e-15)
        if i < 250:
            assert O.sai_angle(t + 0.51 * h) == pytest.approx(t + h, abs=1e-15)
    assert O.sai_angle(-1.0) == pytest.approx(TH_MIN)          # clamped below
    assert O.sai_angle(3.0) == pytest.approx(TH_MAX)           # clamped above
    one = oracle.Geometry(make_config(0), sai_n_theta=1, sai_theta_min=0.05, sai_theta_max=0.3)
    assert one.sai_angle(0.2) == 0.05


def test_pair_factor_at_tabulated_angle():
    """One pair: P_SAI = C G_so G_od T dtheta (1 + cos^2 t_i) cos(t_i / 2) and
    sin(t_i/2) with t_i the nearest tabulated angle; G_so, G_od, dtheta (the
    geometric factors the paper keeps exact, Alg. 2) from 40-digit mpmath."""
    cfg = make_config(0, mask_nx=32, mask_ny=32)
    cfg.mask[:] = 1
    O = sai(cfg, 40)
    mp.mp.dps = 40
    for (iy, iz, ix, jy) in [(0, 0, 0, 0), (3, 5, 7, 9), (7, 7, 15, 15)]:
        pr = O.pair(iy, iz, ix, jy)
        yr = cfg.y_min + (iy + 0.5) * (cfg.y_max - cfg.y_min) / cfg.ny
        zr = cfg.z_min + (iz + 0.5) * (cfg.z_max - cfg.z_min) / cfg.nz
        xd = cfg.det_cx + ((ix + 0.5) - 0.5 * cfg.det_nx) * cfg.det_pitch
        yd = cfg.det_cy + ((jy + 0.5) - 0.5 * cfg.det_ny) * cfg.det_pitch
        r = [mp.mpf(0), mp.mpf(yr), mp.mpf(zr)]
        s = [mp.mpf(xd), mp.mpf(yd) - r[1], mp.mpf(cfg.det_z) - r[2]]
        rn = mp.sqrt(r[1] ** 2 + r[2] ** 2)
        sn = mp.sqrt(sum(x * x for x in s))
        gso = r[2] / rn ** 3
        god = s[2] / sn ** 3
        th = mp.acos((r[1] * s[1] + r[2] * s[2]) / (rn * sn))
        half = mp.mpf(cfg.det_pitch) / 2
        a = [s[0] + half, s[1], s[2]]
        b = [s[0] - half, s[1], s[2]]
        dth = mp.acos(sum(x * y for x, y in zip(a, b)) / (mp.sqrt(sum(x * x for x in a)) * mp.sqrt(sum(x * x for x in b))))
        h = (mp.mpf(TH_MAX) - mp.mpf(TH_MIN)) / 39
        ti = mp.mpf(TH_MIN) + h * mp.floor((th - mp.mpf(TH_MIN)) / h + mp.mpf(0.5))
        P = gso * god * dth * (1 + mp.cos(ti) ** 2) * mp.cos(ti / 2)
        assert pr["P"] == pytest.approx(float(P), rel=1e-11)
        assert pr["sh"] == pytest.approx(float(mp.sin(ti / 2)), rel=1e-13)
        assert pr["theta"] == pytest.approx(float(th), rel=1e-12)  # the pair's own angle is kept


def test_sai_adjoint_identity():
    cfg = make_config(0)
    O = sai(cfg, 250)
    rng = seeded_rng(7, 1)
    for _ in range(5):
        f = rng.uniform(0, 1, O.f_shape)
        w = rng.uniform(0, 1, O.g_shape)
        lhs = float(np.sum(O.forward(f) * w))
        rhs = float(np.sum(f * O.backward(w)))
        assert abs(lhs - rhs) <= 1e-10 * abs(lhs)


def test_sai_error_decreases_with_n_theta():
    """NRMSE (RMSE over the RMS of the exact result) of the SAI
    forward (on the phantom) and backward (on noiseless data, as Table I)
    decreases monotonically in N_theta (SPEC.md:614 AC3), roughly as 1/N for
    nearest-neighbour sampling.  On this config the backward error is also
    below the forward one, as in Table I (0.67 % vs 6.20 %);
    that ordering is data-dependent (not so on config 1)."""
    cfg = make_config(0)
    O = oracle.Geometry(cfg)
    f = cfg.f.astype(np.float64)
    g = O.forward(f)
    b = O.backward(g)
    ef, eb = [], []
    for n in (125, 250, 500, 1000, 2000):
        S = sai(cfg, n)
        ef.append(np.linalg.norm(S.forward(f) - g) / np.linalg.norm(g))
        eb.append(np.linalg.norm(S.backward(g) - b) / np.linalg.norm(b))
    assert all(x > y for x, y in zip(ef, ef[1:])) and all(x > y for x, y in zip(eb, eb[1:]))
    assert ef[-1] < ef[0] / 8  # 16x more angles: ~1/N decay
    assert all(x < y for x, y in zip(eb, ef))


def test_sai_fine_grid_converges_to_exact():
    cfg = make_config(0)
    O = oracle.Geometry(cfg)
    f = cfg.f.astype(np.float64)
    g = O.forward(f)
    S = sai(cfg, 200001)
    assert np.linalg.norm(S.forward(f) - g) / np.linalg.norm(g) < 2e-5
