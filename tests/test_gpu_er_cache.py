"""Energy-resolving operators from the pair cache (er_cache.cu):
lanes-as-energies forward with register sums, fixed-point integer-atomic backward.
Option er_cache=1 (the default runs the direct per-term kernels, operators.cu,
which measured as fast: DESIGN.md 4.3e).  Held to the oracle bar and
cross-checked against the direct kernels, which share none of this code."""
import numpy as np
import pytest

import oracle
from workloads import make_config
from workloads.configs import seeded_rng

torch = pytest.importorskip("torch")
P = pytest.importorskip("paper_1603_06400_b200")

from test_gpu_parity import assert_parity, gpu_backward, gpu_forward, rel_l2, rnd  # noqa: E402

pytestmark = pytest.mark.gpu

SHAPES = [
    {},                                                         # config 0's energy-resolving twin
    dict(ny=6, nz=5, nq=21, det_nx=7, det_ny=19),               # ragged
    dict(ny=9, nz=31, nq=37, det_nx=13, det_ny=29, ne=40, energy_kev=np.linspace(21.0, 149.0, 40),
         phi=np.linspace(1.0, 0.2, 40)),                        # 3 energy rounds, >128-voxel blocks
    dict(energy_kev=np.array([30.0, 33.0, 41.0, 55.0, 60.0, 80.0, 101.0, 119.0])),  # non-uniform: full window
    dict(q_min=0.15, q_max=0.25, nq=9),                         # windows cut by the q grid
    dict(ne=128, energy_kev=np.linspace(20.0, 150.0, 128), phi=np.ones(128)),  # 8 rounds (the maximum)
]


def _desc(over):
    d = make_config(0, energy_resolving=1).desc()
    d.update(over)
    if "energy_kev" in over and "ne" not in over:
        d["ne"] = len(over["energy_kev"])
    return d


@pytest.mark.parametrize("over", SHAPES, ids=range(len(SHAPES)))
def test_er_cache_vs_oracle_and_direct(over):
    d = _desc(over)
    G = P.Geometry(d, options="er_cache=1")
    D = P.Geometry(d)
    O = oracle.Geometry(d)
    assert G.query("er_cache_records") > 0 and D.query("er_cache_records") == 0
    f, w = rnd(G.f_shape, 0, 110), rnd(G.g_shape, 0, 111)
    G.set_timing(True)
    gf, gb = gpu_forward(G, f), gpu_backward(G, w)
    kt = G.kernel_times()
    assert "k_er_fwd" in kt and "k_er_bwd" in kt
    assert_parity(gf, O.forward(f), f"er cache {over} forward")
    assert_parity(gb, O.backward(w), f"er cache {over} backward")
    assert rel_l2(gf, gpu_forward(D, f)) < 1e-6
    assert rel_l2(gb, gpu_backward(D, w)) < 2e-6
    G.set_option("er_fwd", 1)  # the compacted forward k_er_fwd2
    gf2 = gpu_forward(G, f)
    assert_parity(gf2, O.forward(f), f"er cache compacted {over} forward")
    assert rel_l2(gf2, gf) < 1e-6


def test_er_cache_records_are_open_pairs():
    """Every record is an open pair (at most the oracle's open-pair count; only pairs
    whose whole energy window misses the q grid are dropped)."""
    cfg = make_config(0, energy_resolving=1)
    G = P.Geometry(cfg.desc(), options="er_cache=1")
    pairs, open_, terms = oracle.Geometry(cfg).count_terms()
    assert 0 < G.query("er_cache_records") <= open_
    # config 0: every energy of every open pair is in range (test_effective_terms_config0)
    assert G.query("er_cache_records") == open_


def test_er_cache_deterministic_and_wide_range():
    cfg = make_config(0, energy_resolving=1)
    d = cfg.desc()
    d.update(ny=12, nz=10, det_nx=20, det_ny=24)
    G, O = P.Geometry(d, options="er_cache=1"), oracle.Geometry(d)
    f = rnd(G.f_shape, 0, 112)
    w = (10.0 ** seeded_rng(0, 113).uniform(-3, 3, G.g_shape)).astype(np.float32)
    g1, g2 = gpu_forward(G, f), gpu_forward(G, f)
    b1, b2 = gpu_backward(G, w), gpu_backward(G, w)
    assert np.array_equal(g1, g2) and np.array_equal(b1, b2)
    assert_parity(b1, O.backward(w), "er cache backward, log-uniform w")


def test_er_cache_config4_sampled():
    """Config 4 at full size through the pair-cache kernels (sampled outputs)."""
    from test_gpu_parity import _sample
    cfg = make_config(4)
    G, O = P.Geometry(cfg.desc(), options="er_cache=1"), oracle.Geometry(cfg)
    assert G.query("er_cache_records") > 0
    g = gpu_forward(G, cfg.f).reshape(cfg.n_det, cfg.ne)
    pix = _sample(cfg.n_det, 2048, 43)
    ref = O.forward_pixels(cfg.f, pix)
    assert_parity(g[pix], ref, "c4 er-cache forward, 2048 pixels")
    G.set_option("er_fwd", 1)
    g2 = gpu_forward(G, cfg.f).reshape(cfg.n_det, cfg.ne)
    assert_parity(g2[pix], ref, "c4 er-cache compacted forward, 2048 pixels")
    w = rnd(G.g_shape, 4, 10)
    b = gpu_backward(G, w).reshape(cfg.n_vox, cfg.nq)
    vox = _sample(cfg.n_vox, 64, 44)
    assert_parity(b[vox], O.backward_voxels(w, vox), "c4 er-cache backward, 64 voxels")
