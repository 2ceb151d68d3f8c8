"""C-ABI checks that need no GPU: the library loads, exports every symbol the
header declares, and validates descriptors before touching a device."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_1603_06400_b200 as P
from paper_1603_06400_b200 import binding
from workloads import make_config

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    h = open(os.path.join(ROOT, "include", "cacsi.h")).read()
    return sorted(set(re.findall(r"CACSI_API[^;(]*?\b(cacsi_\w+)\s*\(", h)))


def test_header_declares_the_north_star_calls():
    syms = declared_symbols()
    for name in ("cacsi_geometry_create", "cacsi_forward", "cacsi_backward", "cacsi_neg_loglik", "cacsi_iterate"):
        assert name in syms


def test_library_exports_every_declared_symbol():
    lib = P.lib()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert sorted(binding.SYMBOLS) == declared_symbols()


def test_status_strings():
    assert P.status_string(0) == "ok"
    assert P.status_string(2) == "invalid argument"
    assert P.status_string(99) == "unknown status"


def _desc(**over):
    d = make_config(0).desc()
    d.update(over)
    return d


def _create(d, options=None):
    g = binding.GeometryDesc()
    e = np.ascontiguousarray(d["energy_kev"], np.float64)
    ph = np.ascontiguousarray(d["phi"], np.float64)
    m = np.ascontiguousarray(d["mask"], np.uint8)
    for name, _ in binding.GeometryDesc._fields_:
        if name not in ("energy_kev", "phi", "mask"):
            setattr(g, name, d[name])
    g.energy_kev = e.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    g.phi = ph.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    g.mask = m.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))
    h = ctypes.c_void_p()
    st = P.lib().cacsi_geometry_create_ex(ctypes.byref(g), 0, options, ctypes.byref(h))
    if st == 0:
        P.lib().cacsi_geometry_destroy(h)
    return st


@pytest.mark.parametrize("over", [
    dict(ny=0), dict(nq=1), dict(nq=401), dict(ne=300, energy_kev=np.linspace(20, 150, 300), phi=np.ones(300)),
    dict(z_min=-1.0), dict(z_max=900.0), dict(mask_z=1200.0), dict(det_pitch=0.0), dict(mask_pitch=-1.0),
    dict(q_max=0.01), dict(scale=0.0), dict(energy_resolving=2),
    dict(energy_kev=np.array([30, 40, 40, 50, 60, 70, 80, 90.0])),
    dict(phi=-np.ones(8)), dict(y_min=9.0),
    dict(sai_n_theta=-1), dict(sai_n_theta=250, sai_theta_min=0.5, sai_theta_max=0.1),
    dict(sai_n_theta=250, sai_theta_min=0.0, sai_theta_max=4.0),
    dict(sai_n_theta=250, sai_theta_min=-0.1, sai_theta_max=0.5),
    dict(sai_n_theta=250, sai_theta_min=0.01, sai_theta_max=0.5, energy_resolving=1),
    # a pixel too wide for dtheta's series atan(x) = x (1 - x^2/3) (x <= 0.0149)
    dict(det_pitch=20.0), dict(det_z=820.0, mask_z=810.0, det_pitch=7.0),
])
def test_invalid_descriptors_rejected(over):
    assert _create(_desc(**over)) == binding.CACSI_ERR_INVALID


def test_invalid_mask_byte_rejected():
    d = _desc()
    m = d["mask"].copy()
    m[3, 4] = 2
    d["mask"] = m
    assert _create(d) == binding.CACSI_ERR_INVALID


def test_null_pointers():
    L = P.lib()
    assert L.cacsi_geometry_create(None, 0, None) == binding.CACSI_ERR_NULL
    assert L.cacsi_forward(None, None, None, None) == binding.CACSI_ERR_NULL
    assert L.cacsi_backward(None, None, None, None) == binding.CACSI_ERR_NULL
    assert L.cacsi_iterate(None, None, None, None, None, 0.0, 1, None, None) == binding.CACSI_ERR_NULL
    assert L.cacsi_neg_loglik(None, None, None, None, 0.0, None, None, None) == binding.CACSI_ERR_NULL
    assert L.cacsi_workspace_bytes(None) == 0
    L.cacsi_geometry_destroy(None)


def test_no_device_is_an_error_not_a_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    assert _create(_desc()) == binding.CACSI_ERR_CUDA


@pytest.mark.parametrize("args", [(32, 64, 8, 16), (16, 16, 4, 8), (128, 128, 8, 16), (256, 256, 8, 16),
                                  (6, 10, 3, 2), (8, 12, 2, 6), (4, 4, 1, 2)])
def test_symmetric_subsets_match_oracle_partition(args):
    """cacsi_symmetric_subsets (closed-form modular rule, host only) equals the
    oracle's literal MATLAB-list enumeration of PAPER.md:383-387."""
    from oracle import recon
    np.testing.assert_array_equal(binding.symmetric_subsets(*args), recon.symmetric_partition(*args))


@pytest.mark.parametrize("args", [(32, 64, 3, 16), (32, 64, 8, 15), (32, 60, 8, 16), (31, 64, 8, 16),
                                  (32, 64, 0, 16), (32, 64, 8, 0)])
def test_symmetric_subsets_rejects_bad_steps(args):
    with pytest.raises(binding.CacsiError) as ei:
        binding.symmetric_subsets(*args)
    assert ei.value.status == binding.CACSI_ERR_INVALID


@pytest.mark.parametrize("opts", [b"bogus=1", b"pair_cache=2", b"pair_cache", b"=1", b"ts=0,", b"ts=0;direct=1",
                                  b"pcv_budget_kb=1000", b"wgemm=x", b"ts= 0"])
def test_invalid_options_rejected(opts):
    """Kernel-variant options are validated before any device is touched."""
    assert _create(_desc(), opts) == binding.CACSI_ERR_INVALID


@pytest.mark.parametrize("opts", [None, b"", b"pair_cache=0", b"ts=0,direct=1,wgemm=2", b"graphs=0,pcv_items=4"])
def test_valid_options_reach_the_device_check(opts):
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    assert _create(_desc(), opts) == binding.CACSI_ERR_CUDA


def test_library_reads_no_environment():
    """No getenv in the C ABI library (kernel variants are explicit options)."""
    csrc = os.path.join(ROOT, "paper_1603_06400_b200", "csrc")
    for fn in os.listdir(csrc):
        assert "getenv" not in open(os.path.join(csrc, fn)).read(), fn
