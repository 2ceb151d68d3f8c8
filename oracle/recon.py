"""Reconstruction oracle (TEST INFRASTRUCTURE): objective, closed-form update,
Alg. 5.  fp64 numpy, written in the paper's notation (App. B, C).

Readings: R13 quadratic psi(x) = x^2/2 (omega = 1) by default,
Huber psi_delta as the edge-preserving option (R21), 4-connected (y, z)
neighbourhood inside one q bin, w_jk = 1, symmetric (N^b = N); R14 update
edge cases; R15 neg_loglik omits sum ln y! and keeps the paper's
double-counted R; R20 ordered subsets (Alg. 6): row-group-major subset
order, penalty weight beta / P per sub-iteration.
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


class Penalty:
    """Edge-preserving potential psi_delta of Eq. 7 with its
    derivative psi_dot and the surrogate curvature omega(x) = psi_dot(x) / x
    (PAPER.md:686-698).

    kind "quadratic": psi(x) = x^2 / 2 (the default reading R13).
    kind "huber":     psi(x) = x^2 / 2 for |x| <= delta, delta |x| - delta^2 / 2
                      otherwise (Huber 1981, one of the potentials the paper
                      cites at PAPER.md:346; reading R21), omega(0) = 1.
    """

    def __init__(self, kind: str = "quadratic", delta: float = float("inf")):
        assert kind in ("quadratic", "huber")
        if kind == "huber":
            assert delta > 0
        self.kind, self.delta = kind, float(delta)

    def psi(self, x):
        x = np.asarray(x, np.float64)
        if self.kind == "quadratic":
            return 0.5 * x * x
        ax, d = np.abs(x), self.delta
        return np.where(ax <= d, 0.5 * x * x, d * ax - 0.5 * d * d)

    def psi_dot(self, x):
        x = np.asarray(x, np.float64)
        if self.kind == "quadratic":
            return x
        return np.clip(x, -self.delta, self.delta)

    def omega(self, x):
        x = np.asarray(x, np.float64)
        if self.kind == "quadratic":
            return np.ones_like(x)
        ax = np.abs(x)
        with np.errstate(divide="ignore", invalid="ignore"):
            return np.where(ax <= self.delta, 1.0, self.delta / ax)


QUADRATIC = Penalty()


def psi(x):
    return QUADRATIC.psi(x)


def psi_dot(x):
    return QUADRATIC.psi_dot(x)


def omega(x):
    return QUADRATIC.omega(x)


def penalty(f, pen: Penalty = QUADRATIC):
    """R(f) = sum_j sum_{k in N_j} w_jk psi(f_j - f_k)   (each pair counted twice)."""
    f = np.asarray(f, dtype=np.float64)
    R = 0.0
    for fk, valid in _neighbour_shifts(f):
        R += pen.psi(f - fk)[valid].sum()
    return float(R)


def neg_loglik(l, y, r):
    """L = sum_i (l_i + r_i) - y_i ln(l_i + r_i)  (ln y_i! dropped, reading R15)."""
    z = np.asarray(l, np.float64) + np.asarray(r, np.float64)
    y = np.asarray(y, np.float64)
    with np.errstate(divide="ignore", invalid="ignore"):
        ylogz = np.where(y > 0, y * np.log(z), 0.0)
    return float(np.sum(z - ylogz))


def objective(l, y, r, f, beta, pen: Penalty = QUADRATIC):
    """J = L + beta R (Eq. overall_objective)."""
    return neg_loglik(l, y, r) + beta * penalty(f, pen)


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
def update(f_hat, b1, b2, beta, pen: Penalty = QUADRATIC):
    """f^{t+1} from f^t = f_hat, b^(1) = A^T 1, b^(2) = A^T (y / (l + r))."""
    f_hat = np.asarray(f_hat, np.float64)
    b1 = np.asarray(b1, np.float64)
    b2 = np.asarray(b2, np.float64)
    b3 = np.zeros_like(f_hat)
    b5 = np.zeros_like(f_hat)
    for fk, valid in _neighbour_shifts(f_hat):
        # b3 = 2 sum_{k in N_j} w_jk omega(f_j - f_k); b5 = sum w_jk psi_dot(f_j - f_k)
        b3 += np.where(valid, 2.0 * pen.omega(f_hat - fk), 0.0)
        b5 += np.where(valid, pen.psi_dot(f_hat - fk), 0.0)
    b4, b6 = b3, b5  # symmetric neighbourhood: N^b = N, w_jk = w_kj
    chi1 = beta * (b3 + b4)
    chi2 = b1 + beta * (-f_hat * (b3 + b4) + b5 + b6)
    chi3 = f_hat * b2
    out = np.array(lemma_minimizer(chi1, chi2, chi3), dtype=np.float64)
    # reading R14: chi1 = 0 and chi2 <= 0 (voxel never seen, b1 = 0): keep f_hat
    keep = (chi1 <= 0) & (chi2 <= 0)
    out[keep] = f_hat[keep]
    return out


def em_iterate(geom, f0, y, r, b1, beta, n_iter, trace=None, pen: Penalty = QUADRATIC):
    """Alg. 5 with the oracle's fp64 operators.

    Returns the list of iterates [f^1, ..., f^n].  If `trace` is a list, the
    objective J(f^t) for t = 0..n is appended to it."""
    f = np.asarray(f0, np.float64).copy()
    iterates = []
    l = geom.forward(f)
    if trace is not None:
        trace.append(objective(l, y, r, f, beta, pen))
    for _ in range(n_iter):
        rat = ratio(l, y, r)                  # y ./ (A f + r)
        b2 = geom.backward(rat)               # Back_project(y ./ z)
        f = update(f, b1, b2, beta, pen)      # Eq. f_update
        iterates.append(f.copy())
        l = geom.forward(f)
        if trace is not None:
            trace.append(objective(l, y, r, f, beta, pen))
    return iterates


# ---- ordered subsets (Alg. 6; Fig. 6) --------
def symmetric_partition(M: int, N: int, rho_z: int, rho_y: int) -> np.ndarray:
    """Symmetry-preserving measurement-space partition of an M x N detector
    (PAPER.md:383-387), written as the paper's MATLAB index lists (1-based):

      vertical:   rows m:rho_z:M/2 and M-m+1:-rho_z:M/2+1, 1 <= m <= rho_z
      horizontal: columns n:rho_y:N and N-n+1:-rho_y:1,   1 <= n <= rho_y/2

    Subset (m, n) = (row group, column group); P = rho_z rho_y / 2.  Returns
    sub[row][col] in 0..P-1 with p = (m-1) (rho_y/2) + (n-1) (reading R20:
    row-group-major order).  Rows are the paper's vertical (z) index = the
    config frame's det x rows; columns its horizontal (y) index."""
    if M % 2 or (M // 2) % rho_z or rho_y % 2 or N % rho_y or rho_z < 1 or rho_y < 2:
        raise ValueError("partition needs rho_z | M/2, rho_y even, rho_y | N")
    sub = -np.ones((M, N), dtype=np.int64)
    half = rho_y // 2
    for m in range(1, rho_z + 1):
        rows = list(range(m, M // 2 + 1, rho_z)) + list(range(M - m + 1, M // 2, -rho_z))
        for n in range(1, half + 1):
            cols = list(range(n, N + 1, rho_y)) + list(range(N - n + 1, 0, -rho_y))
            for i in rows:
                for j in cols:
                    assert sub[i - 1, j - 1] < 0, "subsets overlap"
                    sub[i - 1, j - 1] = (m - 1) * half + (n - 1)
    assert (sub >= 0).all(), "subsets do not cover the detector"
    return sub


def osem_iterate(geom, f0, y, r, subsets, beta, n_outer, trace=None, pen: Penalty = QUADRATIC,
                 restricted: bool = False):
    """Alg. 6: per outer iteration sweep p = 0..P-1:
    z_p = A_p f + r_p,  b2_p = A_p^T (y_p ./ z_p),  f <- Eq. f_update with
    b1_p = A_p^T 1 and penalty weight beta / P (reading R20: the subset
    data term stands for 1/P of L).  A_p f = (A f) restricted to subset p and
    A_p^T w = A^T (w 1_p) -- the plain definitions; restricted=True evaluates
    the same sums over the subset's pixels only (forward_pixels /
    backward_pixels; pinned equal in tests).  Returns [f^1, ...] (after each
    OUTER iteration); `trace` gets J(f^t) of the FULL objective."""
    sub = np.asarray(subsets).reshape(-1)
    P = int(sub.max()) + 1
    pix = [np.flatnonzero(sub == p) for p in range(P)]
    ind = [(sub == p).astype(np.float64).reshape(geom.g_shape) for p in range(P)]
    ones = np.ones(geom.g_shape)

    def fwd_p(f, p):
        if restricted:
            out = np.zeros(geom.g_shape).reshape(-1)
            out[pix[p]] = geom.forward_pixels(f, pix[p])
            return out.reshape(geom.g_shape)
        return geom.forward(f) * ind[p]

    def bwd_p(w, p):
        return geom.backward_pixels(w, pix[p]) if restricted else geom.backward(w * ind[p])

    b1 = [bwd_p(ones, p) for p in range(P)]
    f = np.asarray(f0, np.float64).copy()
    out = []
    if trace is not None:
        trace.append(objective(geom.forward(f), y, r, f, beta, pen))
    for _ in range(n_outer):
        for p in range(P):
            rat = ratio(fwd_p(f, p), y, r) * ind[p]
            b2 = bwd_p(rat, p)
            f = update(f, b1[p], b2, beta / P, pen)
        out.append(f.copy())
        if trace is not None:
            trace.append(objective(geom.forward(f), y, r, f, beta, pen))
    return out
