"""Brute-force dense system matrix (TEST INFRASTRUCTURE, tiny grids only).

A is assembled element by element from the closed forms of PAPER.md:103-105
and App. A, vectorised over pairs with numpy.  It deliberately uses DIFFERENT
formulas from oracle.c so that it cross-checks the C loops rather than
retyping them:

  * G_so = z / (y^2 + z^2)^1.5          (the simplified form)
  * G_od = s_z / |s|^3                  (|n_d . s^| / s^2 with n_d = z^)
  * theta  = 2 atan2(|r^ - s^|, |r^ + s^|)   (half-angle form; C uses acos)
  * dtheta = 2 atan2(|a^ - b^|, |a^ + b^|)   (C uses atan2(|a x b|, a . b))
  * all Q hat weights Lambda(u_k - j) evaluated (C only evaluates the two
    non-zero ones).

The mask-cell rule (reading R8) is a definition of the discretisation and is
written with the same op order as oracle.c (numpy elementwise ops are
correctly rounded, no FMA), which the exact-tie tests rely on.

Column index: (iy * nz + iz) * nq + j.  Row index: pixel ix * det_ny + jy,
times ne + k in the energy-resolving case.
"""
from __future__ import annotations

import numpy as np

HC = 12.3984193


def _unit(v):
    return v / np.linalg.norm(v, axis=-1, keepdims=True)


def _angle(a, b):
    ua, ub = _unit(a), _unit(b)
    return 2.0 * np.arctan2(np.linalg.norm(ua - ub, axis=-1), np.linalg.norm(ua + ub, axis=-1))


def pair_arrays(d):
    """Per-pair factors for every (pixel, voxel), shape (n_det, n_vox)."""
    ny, nz = d["ny"], d["nz"]
    yv = d["y_min"] + (np.arange(ny) + 0.5) * ((d["y_max"] - d["y_min"]) / ny)
    zv = d["z_min"] + (np.arange(nz) + 0.5) * ((d["z_max"] - d["z_min"]) / nz)
    xd = d["det_cx"] + ((np.arange(d["det_nx"]) + 0.5) - 0.5 * d["det_nx"]) * d["det_pitch"]
    yd = d["det_cy"] + ((np.arange(d["det_ny"]) + 0.5) - 0.5 * d["det_ny"]) * d["det_pitch"]
    YR, ZR = np.meshgrid(yv, zv, indexing="ij")
    YR, ZR = YR.ravel(), ZR.ravel()                     # voxel v = iy * nz + iz
    XD, YD = np.meshgrid(xd, yd, indexing="ij")
    XD, YD = XD.ravel(), YD.ravel()                     # pixel p = ix * det_ny + jy
    zd = d["det_z"]
    nv, npx = YR.size, XD.size
    r = np.stack([np.zeros(nv), YR, ZR], -1)[None, :, :].repeat(npx, 0)
    rp = np.stack([XD, YD, np.full(npx, zd)], -1)[:, None, :].repeat(nv, 1)
    s = rp - r
    gso = ZR / (YR ** 2 + ZR ** 2) ** 1.5
    sn = np.linalg.norm(s, axis=-1)
    god = s[..., 2] / sn ** 3
    th = _angle(r, s)
    half = 0.5 * d["det_pitch"]
    ex = np.array([1.0, 0.0, 0.0])
    dth = _angle(s + half * ex, s - half * ex)
    # mask cell, reading R8 (same op order as the definition)
    t = (d["mask_z"] - ZR[None, :]) / (zd - ZR[None, :])
    px = t * XD[:, None]
    py = YR[None, :] + t * (YD[:, None] - YR[None, :])
    m0x = d["mask_cx"] - (0.5 * d["mask_nx"]) * d["mask_pitch"]
    m0y = d["mask_cy"] - (0.5 * d["mask_ny"]) * d["mask_pitch"]
    fx = np.floor((px - m0x) / d["mask_pitch"])
    fy = np.floor((py - m0y) / d["mask_pitch"])
    inside = (fx >= 0) & (fy >= 0) & (fx < d["mask_nx"]) & (fy < d["mask_ny"])
    mask = np.asarray(d["mask"])
    T = np.zeros(fx.shape)
    T[inside] = mask[fx[inside].astype(int), fy[inside].astype(int)]
    P = d["scale"] * gso[None, :] * god * T * dth * (1.0 + np.cos(th) ** 2) * np.cos(0.5 * th)
    return dict(P=P, theta=th, dtheta=dth, T=T, G_so=np.broadcast_to(gso, P.shape), G_od=god)


def dense_A(d) -> np.ndarray:
    """The system matrix H of the discretised model."""
    d = d.desc() if hasattr(d, "desc") else d
    pa = pair_arrays(d)
    P, th = pa["P"], pa["theta"]
    E = np.asarray(d["energy_kev"], dtype=np.float64)
    phi = np.asarray(d["phi"], dtype=np.float64)
    nq = d["nq"]
    dq = (d["q_max"] - d["q_min"]) / (nq - 1)
    sh = np.sin(0.5 * th)                                   # (npx, nv)
    u = (E[None, None, :] * sh[..., None] / HC - d["q_min"]) / dq   # (npx, nv, ne)
    j = np.arange(nq)
    lam = np.maximum(0.0, 1.0 - np.abs(u[..., None] - j))   # (npx, nv, ne, nq)
    w = (phi * E)[None, None, :, None] * lam * P[..., None, None]
    npx, nv = P.shape
    if d["energy_resolving"]:
        # rows (pixel, k), columns (voxel, j)
        return w.transpose(0, 2, 1, 3).reshape(npx * d["ne"], nv * nq)
    return w.sum(axis=2).reshape(npx, nv * nq)
