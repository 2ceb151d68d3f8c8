"""Thin ctypes binding of libcacsi.so (argument marshalling only).

Every step of the hot path runs in the library's CUDA kernels; this module
only converts torch tensors / numpy arrays to pointers and the current CUDA
stream.  There is no CPU fallback: if libcacsi.so is missing or the device is
not sm_100, calls raise.

Names follow include/cacsi.h: geometry_create, forward, backward, neg_loglik,
iterate (+ *_host end-to-end variants).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# CACSI_CHECKED=1 loads the bounds-checked build (python -m paper_1603_06400_b200.build --checked)
LIB_PATH = os.path.join(_HERE, "libcacsi_checked.so" if os.environ.get("CACSI_CHECKED") == "1" else "libcacsi.so")

CACSI_OK, CACSI_ERR_NULL, CACSI_ERR_INVALID, CACSI_ERR_CUDA, CACSI_ERR_NOMEM = range(5)

SYMBOLS = ["cacsi_geometry_create", "cacsi_geometry_create_ex", "cacsi_set_option", "cacsi_geometry_destroy", "cacsi_workspace_bytes", "cacsi_object_size",
           "cacsi_detector_size", "cacsi_forward", "cacsi_backward", "cacsi_neg_loglik", "cacsi_iterate",
           "cacsi_forward_host", "cacsi_backward_host", "cacsi_iterate_host", "cacsi_last_launch_count",
           "cacsi_status_string", "cacsi_ratio", "cacsi_update", "cacsi_set_timing", "cacsi_kernel_times",
           "cacsi_query", "cacsi_update_ex", "cacsi_iterate_ex", "cacsi_neg_loglik_ex", "cacsi_symmetric_subsets",
           "cacsi_forward_subset", "cacsi_backward_subset", "cacsi_osem"]

CACSI_PENALTY_QUADRATIC, CACSI_PENALTY_HUBER = 0, 1


class CacsiError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        super().__init__(f"{where}: {status_string(status)} (status {status})")


class Penalty(ctypes.Structure):
    """cacsi_penalty (include/cacsi.h): kind 0 quadratic, 1 Huber with scale delta."""
    _fields_ = [("kind", ctypes.c_int32), ("delta", ctypes.c_double)]

    @staticmethod
    def make(kind="quadratic", delta=0.0):
        return Penalty(CACSI_PENALTY_HUBER if kind == "huber" else CACSI_PENALTY_QUADRATIC, float(delta))


def _pen(pen):
    if pen is None:
        return None
    if isinstance(pen, Penalty):
        return ctypes.byref(pen)
    kind, delta = pen
    return ctypes.byref(Penalty.make(kind, delta))


class GeometryDesc(ctypes.Structure):
    """cacsi_geometry_desc (include/cacsi.h)."""
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


_lib = None


def lib():
    """Load libcacsi.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run python -m paper_1603_06400_b200.build")
        L = ctypes.CDLL(LIB_PATH)
        vp, fp = ctypes.c_void_p, ctypes.c_void_p
        L.cacsi_geometry_create.argtypes = [ctypes.POINTER(GeometryDesc), ctypes.c_int, ctypes.POINTER(vp)]
        L.cacsi_geometry_create.restype = ctypes.c_int
        L.cacsi_geometry_create_ex.argtypes = [ctypes.POINTER(GeometryDesc), ctypes.c_int, ctypes.c_char_p,
                                               ctypes.POINTER(vp)]
        L.cacsi_geometry_create_ex.restype = ctypes.c_int
        L.cacsi_set_option.argtypes = [vp, ctypes.c_char_p, ctypes.c_int64]
        L.cacsi_set_option.restype = ctypes.c_int
        L.cacsi_geometry_destroy.argtypes = [vp]
        L.cacsi_geometry_destroy.restype = None
        for n in ("cacsi_workspace_bytes", "cacsi_object_size", "cacsi_detector_size"):
            getattr(L, n).argtypes = [vp]
            getattr(L, n).restype = ctypes.c_size_t
        L.cacsi_forward.argtypes = [vp, fp, fp, vp]
        L.cacsi_backward.argtypes = [vp, fp, fp, vp]
        L.cacsi_neg_loglik.argtypes = [vp, fp, fp, fp, ctypes.c_float, vp, vp, vp]
        L.cacsi_iterate.argtypes = [vp, fp, fp, fp, fp, ctypes.c_float, ctypes.c_int32, vp, vp]
        L.cacsi_ratio.argtypes = [vp, fp, fp, fp, fp, vp]
        L.cacsi_update.argtypes = [vp, fp, fp, fp, ctypes.c_float, fp, vp]
        L.cacsi_forward_host.argtypes = [vp, fp, fp, vp]
        L.cacsi_backward_host.argtypes = [vp, fp, fp, vp]
        L.cacsi_iterate_host.argtypes = [vp, fp, fp, fp, fp, ctypes.c_float, ctypes.c_int32, vp]
        for n in ("cacsi_forward", "cacsi_backward", "cacsi_neg_loglik", "cacsi_iterate", "cacsi_forward_host",
                  "cacsi_ratio", "cacsi_update",
                  "cacsi_backward_host", "cacsi_iterate_host"):
            getattr(L, n).restype = ctypes.c_int
        L.cacsi_last_launch_count.argtypes = [vp]
        L.cacsi_last_launch_count.restype = ctypes.c_int32
        L.cacsi_set_timing.argtypes = [vp, ctypes.c_int32]
        L.cacsi_set_timing.restype = ctypes.c_int
        L.cacsi_kernel_times.argtypes = [vp, ctypes.c_int32, ctypes.POINTER(ctypes.c_char_p),
                                         ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int32)]
        L.cacsi_kernel_times.restype = ctypes.c_int32
        L.cacsi_query.argtypes = [vp, ctypes.c_char_p]
        L.cacsi_query.restype = ctypes.c_int64
        pp = ctypes.POINTER(Penalty)
        i32 = ctypes.c_int32
        L.cacsi_update_ex.argtypes = [vp, fp, fp, fp, ctypes.c_float, pp, fp, vp]
        L.cacsi_iterate_ex.argtypes = [vp, fp, fp, fp, fp, ctypes.c_float, pp, i32, vp, vp]
        L.cacsi_neg_loglik_ex.argtypes = [vp, fp, fp, fp, ctypes.c_float, pp, vp, vp, vp]
        L.cacsi_symmetric_subsets.argtypes = [i32, i32, i32, i32, vp, ctypes.POINTER(i32)]
        L.cacsi_forward_subset.argtypes = [vp, fp, vp, i32, fp, vp]
        L.cacsi_backward_subset.argtypes = [vp, fp, vp, i32, fp, vp]
        L.cacsi_osem.argtypes = [vp, fp, fp, fp, fp, vp, vp, i32, ctypes.c_float, pp, i32, vp, vp]
        for n in ("cacsi_update_ex", "cacsi_iterate_ex", "cacsi_neg_loglik_ex", "cacsi_symmetric_subsets",
                  "cacsi_forward_subset", "cacsi_backward_subset", "cacsi_osem"):
            getattr(L, n).restype = ctypes.c_int
        L.cacsi_status_string.argtypes = [ctypes.c_int]
        L.cacsi_status_string.restype = ctypes.c_char_p
        _lib = L
    return _lib


def status_string(s: int) -> str:
    return lib().cacsi_status_string(s).decode()


def _check(s: int, where: str):
    if s != CACSI_OK:
        raise CacsiError(s, where)


def _ptr(t) -> int:
    """Device pointer of a contiguous fp32 CUDA tensor."""
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float32:
        raise TypeError("expected a float32 CUDA tensor")
    if not t.is_contiguous():
        raise ValueError("tensor must be contiguous")
    return t.data_ptr()


def _iptr(t) -> int:
    """Device pointer of a contiguous int32 CUDA tensor."""
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.int32 or not t.is_contiguous():
        raise TypeError("expected a contiguous int32 CUDA tensor")
    return t.data_ptr()


def symmetric_subsets(det_nx: int, det_ny: int, rho_x: int, rho_y: int) -> np.ndarray:
    """cacsi_symmetric_subsets (host only): subset id per pixel, [det_nx][det_ny]."""
    out = np.empty((det_nx, det_ny), dtype=np.int32)
    n = ctypes.c_int32()
    _check(lib().cacsi_symmetric_subsets(det_nx, det_ny, rho_x, rho_y, out.ctypes.data, ctypes.byref(n)),
           "cacsi_symmetric_subsets")
    assert n.value == int(out.max()) + 1
    return out


def _stream(stream):
    if stream is not None:
        return ctypes.c_void_p(stream)
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _np_f32(a, n, writable=False):
    a = np.asarray(a)
    if a.dtype != np.float32 or not a.flags.c_contiguous or (writable and not a.flags.writeable):
        raise TypeError("expected a C-contiguous float32 numpy array")
    if a.size != n:
        raise ValueError(f"expected {n} elements, got {a.size}")
    return a.ctypes.data


class Geometry:
    """A cacsi_geometry handle.  `desc` is a dict of the descriptor fields
    (workloads.Config.desc()) with numpy arrays energy_kev, phi, mask;
    `options` the kernel-variant options of cacsi_geometry_create_ex, as a
    "key=value,..." string or a dict."""

    def __init__(self, desc: dict, device: int = 0, options=None):
        d = dict(desc)
        d.setdefault("sai_n_theta", 0)
        d.setdefault("sai_theta_min", 0.0)
        d.setdefault("sai_theta_max", 0.0)
        self._e = np.ascontiguousarray(d["energy_kev"], dtype=np.float64)
        self._phi = np.ascontiguousarray(d["phi"], dtype=np.float64)
        self._mask = np.ascontiguousarray(d["mask"], dtype=np.uint8)
        s = GeometryDesc()
        for name, _ in GeometryDesc._fields_:
            if name not in ("energy_kev", "phi", "mask"):
                setattr(s, name, d[name])
        s.energy_kev = self._e.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        s.phi = self._phi.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        s.mask = self._mask.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))
        self._desc = s
        self.handle = ctypes.c_void_p()
        if isinstance(options, dict):
            options = ",".join(f"{k}={int(v)}" for k, v in options.items())
        _check(lib().cacsi_geometry_create_ex(ctypes.byref(s), device, options.encode() if options else None,
                                              ctypes.byref(self.handle)), "cacsi_geometry_create_ex")
        self.device = device
        self.f_shape = (d["ny"], d["nz"], d["nq"])
        self.g_shape = (d["det_nx"], d["det_ny"], d["ne"]) if d["energy_resolving"] else (d["det_nx"], d["det_ny"])
        self.n_obj = lib().cacsi_object_size(self.handle)
        self.n_det = lib().cacsi_detector_size(self.handle)
        self.workspace_bytes = lib().cacsi_workspace_bytes(self.handle)

    def close(self):
        if self.handle:
            lib().cacsi_geometry_destroy(self.handle)
            self.handle = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_option(self, key: str, value: int):
        """cacsi_set_option: select a per-call kernel variant."""
        _check(lib().cacsi_set_option(self.handle, key.encode(), int(value)), "cacsi_set_option")

    def set_timing(self, enable: bool = True):
        _check(lib().cacsi_set_timing(self.handle, int(enable)), "cacsi_set_timing")

    def kernel_times(self) -> dict:
        """{kernel name: (total ms, launches)} since the previous call."""
        n = 64
        names = (ctypes.c_char_p * n)()
        ms = (ctypes.c_double * n)()
        cnt = (ctypes.c_int32 * n)()
        k = lib().cacsi_kernel_times(self.handle, n, names, ms, cnt)
        return {names[i].decode(): (ms[i], cnt[i]) for i in range(k)}

    def query(self, key: str) -> int:
        return lib().cacsi_query(self.handle, key.encode())

    @property
    def last_launch_count(self) -> int:
        return lib().cacsi_last_launch_count(self.handle)

    def _dev(self, t, n, name):
        if t.numel() != n:
            raise ValueError(f"{name}: expected {n} elements, got {t.numel()}")
        return _ptr(t)

    # -- device API (torch CUDA fp32 tensors) --------------------------------
    def forward(self, f, g, stream=None):
        _check(lib().cacsi_forward(self.handle, self._dev(f, self.n_obj, "f"), self._dev(g, self.n_det, "g"),
                                   _stream(stream)), "cacsi_forward")
        return g

    def backward(self, w, b, stream=None):
        _check(lib().cacsi_backward(self.handle, self._dev(w, self.n_det, "w"), self._dev(b, self.n_obj, "b"),
                                    _stream(stream)), "cacsi_backward")
        return b

    def neg_loglik(self, f, y, r, beta, out, ws, stream=None):
        _check(lib().cacsi_neg_loglik(self.handle, self._dev(f, self.n_obj, "f"), self._dev(y, self.n_det, "y"),
                                      self._dev(r, self.n_det, "r"), float(beta), out.data_ptr(), ws.data_ptr(),
                                      _stream(stream)), "cacsi_neg_loglik")
        return out

    def iterate(self, f, y, r, b1, beta, n_iter, ws, stream=None):
        _check(lib().cacsi_iterate(self.handle, self._dev(f, self.n_obj, "f"), self._dev(y, self.n_det, "y"),
                                   self._dev(r, self.n_det, "r"), self._dev(b1, self.n_obj, "b1"), float(beta),
                                   int(n_iter), ws.data_ptr(), _stream(stream)), "cacsi_iterate")
        return f

    def ratio(self, l, y, r, out, stream=None):
        _check(lib().cacsi_ratio(self.handle, self._dev(l, self.n_det, "l"), self._dev(y, self.n_det, "y"),
                                 self._dev(r, self.n_det, "r"), self._dev(out, self.n_det, "ratio"),
                                 _stream(stream)), "cacsi_ratio")
        return out

    def update(self, f_hat, b1, b2, beta, f_new, stream=None):
        _check(lib().cacsi_update(self.handle, self._dev(f_hat, self.n_obj, "f_hat"), self._dev(b1, self.n_obj, "b1"),
                                  self._dev(b2, self.n_obj, "b2"), float(beta), self._dev(f_new, self.n_obj, "f_new"),
                                  _stream(stream)), "cacsi_update")
        return f_new

    # -- penalties (Huber) and ordered subsets (Alg. 6) ---------------------
    def update_ex(self, f_hat, b1, b2, beta, pen, f_new, stream=None):
        _check(lib().cacsi_update_ex(self.handle, self._dev(f_hat, self.n_obj, "f_hat"),
                                     self._dev(b1, self.n_obj, "b1"), self._dev(b2, self.n_obj, "b2"), float(beta),
                                     _pen(pen), self._dev(f_new, self.n_obj, "f_new"), _stream(stream)),
               "cacsi_update_ex")
        return f_new

    def iterate_ex(self, f, y, r, b1, beta, pen, n_iter, ws, stream=None):
        _check(lib().cacsi_iterate_ex(self.handle, self._dev(f, self.n_obj, "f"), self._dev(y, self.n_det, "y"),
                                      self._dev(r, self.n_det, "r"), self._dev(b1, self.n_obj, "b1"), float(beta),
                                      _pen(pen), int(n_iter), ws.data_ptr(), _stream(stream)), "cacsi_iterate_ex")
        return f

    def neg_loglik_ex(self, f, y, r, beta, pen, out, ws, stream=None):
        _check(lib().cacsi_neg_loglik_ex(self.handle, self._dev(f, self.n_obj, "f"), self._dev(y, self.n_det, "y"),
                                         self._dev(r, self.n_det, "r"), float(beta), _pen(pen), out.data_ptr(),
                                         ws.data_ptr(), _stream(stream)), "cacsi_neg_loglik_ex")
        return out

    def forward_subset(self, f, pixels, g, stream=None):
        _check(lib().cacsi_forward_subset(self.handle, self._dev(f, self.n_obj, "f"), _iptr(pixels), pixels.numel(),
                                          self._dev(g, self.n_det, "g"), _stream(stream)), "cacsi_forward_subset")
        return g

    def backward_subset(self, w, pixels, b, stream=None):
        _check(lib().cacsi_backward_subset(self.handle, self._dev(w, self.n_det, "w"), _iptr(pixels),
                                           pixels.numel(), self._dev(b, self.n_obj, "b"), _stream(stream)),
               "cacsi_backward_subset")
        return b

    def osem(self, f, y, r, b1_subsets, pixels, offsets, beta, pen, n_outer, ws, stream=None):
        """offsets: host int sequence of length P + 1; b1_subsets: [P, *f_shape] fp32 CUDA."""
        off = np.ascontiguousarray(offsets, dtype=np.int32)
        P = len(off) - 1
        _check(lib().cacsi_osem(self.handle, self._dev(f, self.n_obj, "f"), self._dev(y, self.n_det, "y"),
                                self._dev(r, self.n_det, "r"), self._dev(b1_subsets, P * self.n_obj, "b1_subsets"),
                                _iptr(pixels), off.ctypes.data, P, float(beta), _pen(pen), int(n_outer),
                                ws.data_ptr(), _stream(stream)), "cacsi_osem")
        return f

    # -- host API (numpy fp32, end-to-end) -----------------------------------
    def forward_host(self, f, g, stream=None):
        _check(lib().cacsi_forward_host(self.handle, _np_f32(f, self.n_obj), _np_f32(g, self.n_det, True),
                                        _stream(stream)),
               "cacsi_forward_host")
        return g

    def backward_host(self, w, b, stream=None):
        _check(lib().cacsi_backward_host(self.handle, _np_f32(w, self.n_det), _np_f32(b, self.n_obj, True),
                                         _stream(stream)),
               "cacsi_backward_host")
        return b

    def iterate_host(self, f, y, r, b1, beta, n_iter, stream=None):
        _check(lib().cacsi_iterate_host(self.handle, _np_f32(f, self.n_obj, True), _np_f32(y, self.n_det),
                                        _np_f32(r, self.n_det), _np_f32(b1, self.n_obj),
                                        float(beta), int(n_iter), _stream(stream)), "cacsi_iterate_host")
        return f


def geometry_create(desc: dict, device: int = 0, options=None) -> Geometry:
    return Geometry(desc, device, options)
