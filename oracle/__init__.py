"""fp64 CPU oracle of arXiv 1603.06400's forward/backward models and Alg. 5.

TEST INFRASTRUCTURE.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package.  It shares no
code with the CUDA path (paper_1603_06400_b200/) and never imports it.

Pieces:
  * oracle.c (ctypes): the dense double sums g = A f, b = A^T w (Alg. 1 / Alg. 3
    loop structure) in the energy form, per-pair
    factors, work counts.
  * dense_A (numpy): the system matrix assembled element by element from the
    closed forms with DIFFERENT angle formulas (half-angle atan2) -- a
    brute-force cross-check of the C loops on tiny grids.
  * recon.py: Lemma 1, the closed-form update (Eq. f_update), the objective
    J = L + beta R and Alg. 5.

Parity status per function is listed in DESIGN.md "Oracle pins".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HC = 12.3984193  # keV Angstrom

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so (gcc -O2 -fopenmp -ffp-contract=off)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared", "-std=c11",
               "-Wall", _SRC, "-o", _LIB + ".tmp", "-lm"]
        subprocess.run(cmd, check=True)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


class _Desc(ctypes.Structure):
    _fields_ = [
        ("ny", ctypes.c_int32), ("nz", ctypes.c_int32),
        ("y_min", ctypes.c_double), ("y_max", ctypes.c_double),
        ("z_min", ctypes.c_double), ("z_max", ctypes.c_double),
        ("nq", ctypes.c_int32), ("q_min", ctypes.c_double), ("q_max", ctypes.c_double),
        ("ne", ctypes.c_int32),
        ("energy_kev", ctypes.POINTER(ctypes.c_double)), ("phi", ctypes.POINTER(ctypes.c_double)),
        ("mask_nx", ctypes.c_int32), ("mask_ny", ctypes.c_int32),
        ("mask_z", ctypes.c_double), ("mask_pitch", ctypes.c_double),
        ("mask_cx", ctypes.c_double), ("mask_cy", ctypes.c_double),
        ("mask", ctypes.POINTER(ctypes.c_uint8)),
        ("det_nx", ctypes.c_int32), ("det_ny", ctypes.c_int32),
        ("det_z", ctypes.c_double), ("det_pitch", ctypes.c_double),
        ("det_cx", ctypes.c_double), ("det_cy", ctypes.c_double),
        ("energy_resolving", ctypes.c_int32), ("scale", ctypes.c_double),
        ("sai_n_theta", ctypes.c_int32), ("sai_theta_min", ctypes.c_double), ("sai_theta_max", ctypes.c_double),
    ]


def _L():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.POINTER
        dp = P(ctypes.c_double)
        i64p = P(ctypes.c_int64)
        lib.oracle_forward.argtypes = [P(_Desc), dp, dp]
        lib.oracle_backward.argtypes = [P(_Desc), dp, dp]
        lib.oracle_forward_pixels.argtypes = [P(_Desc), dp, ctypes.c_long, i64p, dp]
        lib.oracle_backward_voxels.argtypes = [P(_Desc), dp, ctypes.c_long, i64p, dp]
        lib.oracle_backward_pixels.argtypes = [P(_Desc), dp, ctypes.c_long, i64p, dp]
        lib.oracle_pair.argtypes = [P(_Desc), ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, dp]
        lib.oracle_mask_cell.argtypes = [P(_Desc), ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                         ctypes.c_double, P(ctypes.c_int), P(ctypes.c_int)]
        lib.oracle_count_terms.argtypes = [P(_Desc), ctypes.c_long, i64p, i64p]
        lib.oracle_voxel_centre.argtypes = [P(_Desc), ctypes.c_int, ctypes.c_int, dp]
        lib.oracle_det_centre.argtypes = [P(_Desc), ctypes.c_int, ctypes.c_int, dp]
        lib.oracle_sai_angle.argtypes = [P(_Desc), ctypes.c_double]
        lib.oracle_sai_angle.restype = ctypes.c_double
        for fn in ("oracle_G_so", "oracle_G_od"):
            getattr(lib, fn).argtypes = [dp]
            getattr(lib, fn).restype = ctypes.c_double
        lib.oracle_theta.argtypes = [dp, dp]
        lib.oracle_theta.restype = ctypes.c_double
        lib.oracle_dtheta.argtypes = [dp, dp, ctypes.c_double]
        lib.oracle_dtheta.restype = ctypes.c_double
        _lib = lib
    return _lib


class Geometry:
    """Holds an oracle descriptor and keeps its arrays alive."""

    def __init__(self, cfg, **override):
        d = cfg.desc() if hasattr(cfg, "desc") else dict(cfg)
        d.update(override)
        d.setdefault("sai_n_theta", 0)
        d.setdefault("sai_theta_min", 0.0)
        d.setdefault("sai_theta_max", 0.0)
        self.d = d
        self._e = np.ascontiguousarray(d["energy_kev"], dtype=np.float64)
        self._phi = np.ascontiguousarray(d["phi"], dtype=np.float64)
        self._mask = np.ascontiguousarray(d["mask"], dtype=np.uint8)
        assert self._mask.shape == (d["mask_nx"], d["mask_ny"])
        assert self._e.size == d["ne"] and self._phi.size == d["ne"]
        s = _Desc()
        for name, _ in _Desc._fields_:
            if name in ("energy_kev", "phi", "mask"):
                continue
            setattr(s, name, d[name])
        s.energy_kev = self._e.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        s.phi = self._phi.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        s.mask = self._mask.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))
        self.s = s
        self.ny, self.nz, self.nq, self.ne = d["ny"], d["nz"], d["nq"], d["ne"]
        self.det_nx, self.det_ny = d["det_nx"], d["det_ny"]
        self.energy_resolving = int(d["energy_resolving"])

    @property
    def f_shape(self):
        return (self.ny, self.nz, self.nq)

    @property
    def g_shape(self):
        return (self.det_nx, self.det_ny, self.ne) if self.energy_resolving else (self.det_nx, self.det_ny)

    # -- operators ---------------------------------------------------------
    def forward(self, f) -> np.ndarray:
        f = np.ascontiguousarray(f, dtype=np.float64).reshape(self.f_shape)
        g = np.zeros(self.g_shape)
        _L().oracle_forward(ctypes.byref(self.s), _dp(f), _dp(g))
        return g

    def backward(self, w) -> np.ndarray:
        w = np.ascontiguousarray(w, dtype=np.float64).reshape(self.g_shape)
        b = np.zeros(self.f_shape)
        _L().oracle_backward(ctypes.byref(self.s), _dp(w), _dp(b))
        return b

    def forward_pixels(self, f, pix) -> np.ndarray:
        """g at flat pixel indices pix (ix * det_ny + jy); shape (n,) or (n, ne)."""
        f = np.ascontiguousarray(f, dtype=np.float64).reshape(self.f_shape)
        pix = np.ascontiguousarray(pix, dtype=np.int64)
        nout = self.ne if self.energy_resolving else 1
        out = np.zeros((pix.size, nout))
        _L().oracle_forward_pixels(ctypes.byref(self.s), _dp(f), pix.size, _ip(pix), _dp(out))
        return out if self.energy_resolving else out[:, 0]

    def backward_voxels(self, w, vox) -> np.ndarray:
        """b rows at flat voxel indices vox (iy * nz + iz); shape (n, nq)."""
        w = np.ascontiguousarray(w, dtype=np.float64).reshape(self.g_shape)
        vox = np.ascontiguousarray(vox, dtype=np.int64)
        out = np.zeros((vox.size, self.nq))
        _L().oracle_backward_voxels(ctypes.byref(self.s), _dp(w), vox.size, _ip(vox), _dp(out))
        return out

    def backward_pixels(self, w, pix) -> np.ndarray:
        """A_p^T w: the backward sum restricted to flat pixel indices pix (Alg. 6)."""
        w = np.ascontiguousarray(w, dtype=np.float64).reshape(self.g_shape)
        pix = np.ascontiguousarray(pix, dtype=np.int64)
        b = np.zeros(self.f_shape)
        _L().oracle_backward_pixels(ctypes.byref(self.s), _dp(w), pix.size, _ip(pix), _dp(b))
        return b

    def sai_angle(self, theta: float) -> float:
        """The tabulated angle scatter-angle interpolation uses for theta."""
        return _L().oracle_sai_angle(ctypes.byref(self.s), float(theta))

    def pair(self, iy, iz, ix, jy) -> dict:
        out = np.zeros(8)
        _L().oracle_pair(ctypes.byref(self.s), iy, iz, ix, jy, _dp(out))
        keys = ["P", "sh", "ch", "theta", "dtheta", "T", "G_so", "G_od"]
        return dict(zip(keys, out.tolist()))

    def mask_cell(self, y_r, z_r, x_d, y_d):
        cx, cy = ctypes.c_int(), ctypes.c_int()
        inside = _L().oracle_mask_cell(ctypes.byref(self.s), y_r, z_r, x_d, y_d,
                                       ctypes.byref(cx), ctypes.byref(cy))
        return bool(inside), cx.value, cy.value

    def count_terms(self, pix=None):
        """(pairs, open pairs, effective terms) over the given pixels (default all)."""
        if pix is None:
            pix = np.arange(self.det_nx * self.det_ny)
        pix = np.ascontiguousarray(pix, dtype=np.int64)
        out = np.zeros(3, dtype=np.int64)
        _L().oracle_count_terms(ctypes.byref(self.s), pix.size, _ip(pix), _ip(out))
        return tuple(int(v) for v in out)

    def voxel_centre(self, iy, iz):
        """(y, z) of voxel (iy, iz) as oracle.c computes it (reading R9)."""
        out = np.zeros(2)
        _L().oracle_voxel_centre(ctypes.byref(self.s), iy, iz, _dp(out))
        return tuple(out.tolist())

    def det_centre(self, ix, jy):
        """(x, y) of detector pixel (ix, jy) as oracle.c computes it (reading R9)."""
        out = np.zeros(2)
        _L().oracle_det_centre(ctypes.byref(self.s), ix, jy, _dp(out))
        return tuple(out.tolist())

    # -- centres (reading R9), for tests ------------------------------------
    def voxel_centres(self):
        d = self.d
        yp = (d["y_max"] - d["y_min"]) / d["ny"]
        zp = (d["z_max"] - d["z_min"]) / d["nz"]
        y = d["y_min"] + (np.arange(d["ny"]) + 0.5) * yp
        z = d["z_min"] + (np.arange(d["nz"]) + 0.5) * zp
        return y, z

    def det_centres(self):
        d = self.d
        x = d["det_cx"] + ((np.arange(d["det_nx"]) + 0.5) - 0.5 * d["det_nx"]) * d["det_pitch"]
        y = d["det_cy"] + ((np.arange(d["det_ny"]) + 0.5) - 0.5 * d["det_ny"]) * d["det_pitch"]
        return x, y


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _ip(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


# -- single-point factor functions (config frame) ----------------------------
def G_so(r):
    return _L().oracle_G_so(_dp(np.ascontiguousarray(r, dtype=np.float64)))


def G_od(s):
    return _L().oracle_G_od(_dp(np.ascontiguousarray(s, dtype=np.float64)))


def theta(r, rp):
    return _L().oracle_theta(_dp(np.ascontiguousarray(r, dtype=np.float64)),
                             _dp(np.ascontiguousarray(rp, dtype=np.float64)))


def dtheta(r, rp, pitch):
    return _L().oracle_dtheta(_dp(np.ascontiguousarray(r, dtype=np.float64)),
                              _dp(np.ascontiguousarray(rp, dtype=np.float64)), float(pitch))


from .dense import dense_A  # noqa: E402,F401
from . import recon  # noqa: E402,F401
