"""Reconstruction oracle (TEST INFRASTRUCTURE): objective, closed-form update,
Alg. 5.  fp64 numpy, written in the paper's notation (App. B, C).

Readings: R13 quadratic psi(x) = x^2/2 (omega = 1), 4-connected
(y, z) neighbourhood inside one q bin, w_jk = 1, symmetric (N^b = N);
R14 update edge cases; R15 neg_loglik omits sum ln y! and keeps the paper's
double-counted R.
"""
from __future__ import annotations

import numpy as np


# ---- Lemma 1 --------------------------------------------
def lemma_minimizer(a, b, c):
    """argmin_{x in [0, inf]} 1/2 a x^2 + b x - c ln x (+ d), a >= 0, c >= 0.

    a > 0: x* = (-b + sqrt(b^2 + 4ac)) / (2a).  Evaluated as the same number
    written 2c / (b + sqrt(b^2 + 4ac)) when b > 0 (multiply numerator and
    denominator by b + sqrt(D)), which avoids cancellation in fp64.
    a = 0, b > 0: c / b.   a = 0, b <= 0: +inf.
    """
    a, b, c = np.broadcast_arrays(np.asarray(a, float), np.asarray(b, float), np.asarray(c, float))
    out = np.empty(a.shape)
    D = b * b + 4.0 * a * c
    sq = np.sqrt(np.maximum(D, 0.0))
    pos = a > 0
    with np.errstate(divide="ignore", invalid="ignore"):
        textbook = (-b + sq) / (2.0 * a)
        rational = 2.0 * c / (b + sq)
        root = np.where(b > 0, rational, textbook)
        out[pos] = root[pos]
        lin = (~pos) & (b > 0)
        out[lin] = (c / b)[lin]
    out[(~pos) & (b <= 0)] = np.inf
    return out if out.shape else float(out)


# ---- neighbourhood and penalty (Eq. 7) -------------------
def _neighbour_shifts(f):
    """Yield (f_k aligned to f_j, valid mask) for the 4 (y, z) neighbours."""
    ny, nz = f.shape[0], f.shape[1]
    for axis, step in ((0, 1), (0, -1), (1, 1), (1, -1)):
        fk = np.zeros_like(f)
        valid = np.zeros(f.shape[:2], dtype=bool)
        n = f.shape[axis]
        src = [slice(None)] * f.ndim
        dst = [slice(None)] * f.ndim
        if step == 1:
            dst[axis], src[axis] = slice(0, n - 1), slice(1, n)
        else:
            dst[axis], src[axis] = slice(1, n), slice(0, n - 1)
        fk[tuple(dst)] = f[tuple(src)]
        valid[tuple(dst[:2])] = True
        yield fk, valid[:, :, None] & np.ones((1, 1, f.shape[2]), dtype=bool)
    _ = ny, nz


def psi(x):
    return 0.5 * x * x


def psi_dot(x):
    return x


def omega(x):
    return np.ones_like(x)


def penalty(f):
    """R(f) = sum_j sum_{k in N_j} w_jk psi(f_j - f_k)   (each pair counted twice)."""
    f = np.asarray(f, dtype=np.float64)
    R = 0.0
    for fk, valid in _neighbour_shifts(f):
        R += psi(f - fk)[valid].sum()
    return float(R)


def neg_loglik(l, y, r):
    """L = sum_i (l_i + r_i) - y_i ln(l_i + r_i)  (ln y_i! dropped, reading R15)."""
    z = np.asarray(l, np.float64) + np.asarray(r, np.float64)
    y = np.asarray(y, np.float64)
    with np.errstate(divide="ignore", invalid="ignore"):
        ylogz = np.where(y > 0, y * np.log(z), 0.0)
    return float(np.sum(z - ylogz))


def objective(l, y, r, f, beta):
    """J = L + beta R (Eq. overall_objective)."""
    return neg_loglik(l, y, r) + beta * penalty(f)


def ratio(l, y, r, eps=1e-12):
    """y / (l + r); 0 where y = 0 and l + r = 0; y / eps where l + r = 0 < y."""
    z = np.asarray(l, np.float64) + np.asarray(r, np.float64)
    y = np.asarray(y, np.float64)
    out = np.zeros_like(z)
    pos = z > 0
    out[pos] = y[pos] / z[pos]
    out[(~pos) & (y > 0)] = y[(~pos) & (y > 0)] / eps
    return out


# ---- closed-form update (Eq. f_update) -------------------
def update(f_hat, b1, b2, beta):
    """f^{t+1} from f^t = f_hat, b^(1) = A^T 1, b^(2) = A^T (y / (l + r))."""
    f_hat = np.asarray(f_hat, np.float64)
    b1 = np.asarray(b1, np.float64)
    b2 = np.asarray(b2, np.float64)
    b3 = np.zeros_like(f_hat)
    b5 = np.zeros_like(f_hat)
    for fk, valid in _neighbour_shifts(f_hat):
        # b3 = 2 sum_{k in N_j} w_jk omega(f_j - f_k); b5 = sum w_jk psi_dot(f_j - f_k)
        b3 += np.where(valid, 2.0 * omega(f_hat - fk), 0.0)
        b5 += np.where(valid, psi_dot(f_hat - fk), 0.0)
    b4, b6 = b3, b5  # symmetric neighbourhood: N^b = N, w_jk = w_kj
    chi1 = beta * (b3 + b4)
    chi2 = b1 + beta * (-f_hat * (b3 + b4) + b5 + b6)
    chi3 = f_hat * b2
    out = np.array(lemma_minimizer(chi1, chi2, chi3), dtype=np.float64)
    # reading R14: chi1 = 0 and chi2 <= 0 (voxel never seen, b1 = 0): keep f_hat
    keep = (chi1 <= 0) & (chi2 <= 0)
    out[keep] = f_hat[keep]
    return out


def em_iterate(geom, f0, y, r, b1, beta, n_iter, trace=None):
    """Alg. 5 with the oracle's fp64 operators.

    Returns the list of iterates [f^1, ..., f^n].  If `trace` is a list, the
    objective J(f^t) for t = 0..n is appended to it."""
    f = np.asarray(f0, np.float64).copy()
    iterates = []
    l = geom.forward(f)
    if trace is not None:
        trace.append(objective(l, y, r, f, beta))
    for _ in range(n_iter):
        rat = ratio(l, y, r)                  # y ./ (A f + r)
        b2 = geom.backward(rat)               # Back_project(y ./ z)
        f = update(f, b1, b2, beta)           # Eq. f_update
        iterates.append(f.copy())
        l = geom.forward(f)
        if trace is not None:
            trace.append(objective(l, y, r, f, beta))
    return iterates
