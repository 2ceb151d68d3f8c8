"""The direct energy-resolving forward with register accumulators (option er_fwd_reg=1, the
default; csrc/operators.cu k_forward_reg): the oracle bar on energy counts that select each
register-array size, and agreement with the shared-memory-accumulator kernel (er_fwd_reg=0,
the (mid, slope) table form) to well inside the bar; the fixed-point backward."""
import numpy as np
import pytest

import oracle
from workloads import make_config

torch = pytest.importorskip("torch")
P = pytest.importorskip("paper_1603_06400_b200")

from test_gpu_parity import assert_parity, gpu_backward, gpu_forward, rel_l2, rnd  # noqa: E402
from workloads.configs import seeded_rng  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("ne", [8, 17, 40, 64, 100, 128])
def test_er_forward_registers_bitwise_and_oracle(ne):
    d = make_config(0, energy_resolving=1).desc()
    d.update(ne=ne, energy_kev=np.linspace(21.0, 149.0, ne), phi=np.linspace(1.0, 0.3, ne),
             ny=6, nz=5, nq=21, det_nx=7, det_ny=19)
    G = P.Geometry(d)
    assert G.query("er_fcache_records") > 0  # the default forward is the record-fed k_forward_rec
    f = rnd(G.f_shape, 0, 140)
    g1 = gpu_forward(G, f)
    # record-fed vs per-lane mask tests and pair geometry (k_forward_lane): same sums, same order
    G.set_option("er_fwd_rec", 0)
    assert np.array_equal(gpu_forward(G, f), g1)
    # per-lane voxel streams vs warp-uniform voxels: same sums, same order
    G.set_option("er_fwd_lane", 0)
    assert np.array_equal(gpu_forward(G, f), g1)
    G.set_option("er_fwd_reg", 0)
    g0 = gpu_forward(G, f)
    assert_parity(g1, g0, f"er forward registers vs shared accumulators ne={ne}", l2=1e-6, mr=1e-5)
    assert_parity(g1, oracle.Geometry(d).forward(f), f"er forward registers ne={ne}")


@pytest.mark.parametrize("shape", [
    dict(ny=37, nz=41, det_nx=13, det_ny=29, ne=40),   # 2 splits, ragged chunks and pixel tile
    dict(ny=64, nz=67, det_nx=9, det_ny=15, ne=100),   # 5 splits of 896 voxels, 135 pixels
    dict(ny=3, nz=11, det_nx=40, det_ny=7, ne=17),     # one chunk, 280 pixels
])
def test_er_forward_records_multichunk(shape):
    """k_forward_rec over many table chunks (two in flight, lanes running ahead into the next),
    several voxel splits and ragged ends: bit-identical to k_forward_lane and k_forward_reg, and
    the oracle bar."""
    ne = shape["ne"]
    d = make_config(0, energy_resolving=1).desc()
    d.update(energy_kev=np.linspace(21.0, 149.0, ne), phi=np.linspace(1.0, 0.3, ne), nq=33, **shape)
    G = P.Geometry(d)
    assert G.query("er_fcache_records") > 0
    f = rnd(G.f_shape, 0, 142)
    g1 = gpu_forward(G, f)
    assert np.array_equal(gpu_forward(G, f), g1)
    G.set_option("er_fwd_rec", 0)
    assert np.array_equal(gpu_forward(G, f), g1)
    G.set_option("er_fwd_lane", 0)
    assert np.array_equal(gpu_forward(G, f), g1)
    assert_parity(g1, oracle.Geometry(d).forward(f), f"er forward records {shape}")


def test_er_forward_records_off():
    """er_fcache=0 at create: no records, the forward falls back to k_forward_lane (same bits)."""
    d = make_config(0, energy_resolving=1).desc()
    G = P.Geometry(d)
    G0 = P.Geometry(d, options="er_fcache=0")
    assert G0.query("er_fcache_records") == 0
    f = rnd(G.f_shape, 0, 143)
    assert np.array_equal(gpu_forward(G, f), gpu_forward(G0, f))


def test_er_forward_registers_non_uniform_energies():
    d = make_config(0, energy_resolving=1).desc()
    d.update(energy_kev=np.array([30.0, 33.0, 41.0, 55.0, 60.0, 80.0, 101.0, 119.0]))
    G = P.Geometry(d)
    f = rnd(G.f_shape, 0, 141)
    g1 = gpu_forward(G, f)
    G.set_option("er_fwd_reg", 0)
    assert_parity(g1, gpu_forward(G, f), "er forward registers vs shared accumulators, non-uniform", l2=1e-6, mr=1e-5)
    assert_parity(g1, oracle.Geometry(d).forward(f), "er forward registers, non-uniform energies")



# ---- fixed-point energy-resolving backward (option er_bwd_fx=1, the default; k_backward_er_x) ----
def _er_desc(**over):
    d = make_config(0, energy_resolving=1).desc()
    d.update(over)
    return d


ER_BWD_SHAPES = [
    {},
    dict(ne=17, energy_kev=np.linspace(21.0, 149.0, 17), phi=np.linspace(1.0, 0.3, 17), ny=6, nz=5, nq=21,
         det_nx=7, det_ny=19),
    dict(ne=100, energy_kev=np.linspace(21.0, 149.0, 100), phi=np.linspace(1.0, 0.3, 100), ny=5, nz=7, nq=33,
         det_nx=9, det_ny=23),
    dict(ne=128, energy_kev=np.linspace(21.0, 149.0, 128), phi=np.linspace(1.0, 0.3, 128)),
    dict(energy_kev=np.array([30.0, 33.0, 41.0, 55.0, 60.0, 80.0, 101.0, 119.0])),
    dict(q_min=0.15, q_max=0.25, nq=9),
    dict(q_min=0.0, q_max=0.9, nq=40),
]


@pytest.mark.parametrize("si", range(len(ER_BWD_SHAPES)))
def test_er_backward_fixed_point_oracle(si):
    """Every output against the oracle, and against the fp32-histogram kernel (er_bwd_fx=0)
    as an independent GPU cross-check; deterministic bits."""
    d = _er_desc(**ER_BWD_SHAPES[si])
    G = P.Geometry(d)
    w = rnd(G.g_shape, 0, 150 + si)
    b1 = gpu_backward(G, w)
    assert np.array_equal(b1, gpu_backward(G, w))
    assert_parity(b1, oracle.Geometry(d).backward(w), f"er backward fixed point {si}")
    G.set_option("er_bwd_fx", 0)
    b0 = gpu_backward(G, w)
    assert_parity(b1, b0, f"er backward fixed point vs fp32 histograms {si}")


@pytest.mark.parametrize("kind", ["log_uniform", "signed", "ones"])
def test_er_backward_fixed_point_weights(kind):
    """The per-voxel scale follows max |w|: weights over six decades, signed weights
    (bar against the absolute-value operator, reading R19b), and w = 1 (the create-time
    bound measurement's own input)."""
    d = _er_desc(ny=6, nz=5, nq=21, det_nx=7, det_ny=19)
    G, O = P.Geometry(d), oracle.Geometry(d)
    rng = seeded_rng(0, 160)
    if kind == "log_uniform":
        w = (10.0 ** rng.uniform(-3, 3, G.g_shape)).astype(np.float32)
    elif kind == "signed":
        w = rng.uniform(-1, 1, G.g_shape).astype(np.float32)
    else:
        w = np.ones(G.g_shape, np.float32)
    b = gpu_backward(G, w)
    ref = O.backward(w.astype(np.float64))
    if kind != "signed":
        assert_parity(b, ref, f"er backward fixed point, {kind} w")
        return
    absref = O.backward(np.abs(w).astype(np.float64))
    sel = absref >= 1e-3 * absref.max()
    err = np.abs(b - ref)[sel] / absref[sel]
    print(f"er backward fixed point, signed w: rel_l2={rel_l2(b, ref):.3e} max_err_vs_abs={err.max():.3e}")
    assert rel_l2(b, ref) <= 1e-5 and err.max() <= 1e-4


def test_er_backward_fixed_point_zero_and_outliers():
    """w = 0 gives exact zeros; huge weights (the ratio guard's y / 1e-12) on pixels that no
    open pair reaches never deposit, so they must not set the fixed-point scale."""
    d = _er_desc()
    m = d["mask"].copy()
    m[:12, :] = 0
    m[17:, :] = 0
    d["mask"] = m
    G, O = P.Geometry(d), oracle.Geometry(d)
    assert not np.any(gpu_backward(G, np.zeros(G.g_shape, np.float32)))
    n_det = d["det_nx"] * d["det_ny"]
    unseen = np.flatnonzero(np.array([O.count_terms([q])[1] for q in range(n_det)]) == 0)
    assert 0 < unseen.size < n_det
    w = rnd(G.g_shape, 0, 161).reshape(n_det, -1)
    ref = O.backward(w.reshape(G.g_shape).astype(np.float64))
    w[unseen] = np.float32(3e12)
    assert_parity(gpu_backward(G, w.reshape(G.g_shape)), ref, "er backward fixed point, unseen-pixel outliers")


def test_er_backward_fixed_point_config4_sampled():
    """Config 4 at full size: sampled voxels against the oracle, plus the fp32-histogram kernel;
    the forward's per-lane voxel streams against warp-uniform voxels (bitwise)."""
    cfg = make_config(4)
    G, O = P.Geometry(cfg.desc()), oracle.Geometry(cfg.desc())
    g1 = gpu_forward(G, cfg.f)
    G.set_option("er_fwd_lane", 0)
    assert np.array_equal(gpu_forward(G, cfg.f), g1)
    G.set_option("er_fwd_lane", 1)
    w = rnd(G.g_shape, 4, 162)
    b = gpu_backward(G, w).reshape(cfg.n_vox, cfg.nq)
    rng = np.random.default_rng(4)
    vox = np.unique(np.concatenate([rng.choice(cfg.n_vox, 6, replace=False), [0, cfg.n_vox - 1]]))
    assert_parity(b[vox], O.backward_voxels(w, vox), "c4 er backward fixed point sampled")
    G.set_option("er_bwd_fx", 0)
    b0 = gpu_backward(G, w).reshape(cfg.n_vox, cfg.nq)
    assert_parity(b, b0, "c4 er backward fixed point vs fp32 histograms (every voxel)")
    # the voxel-major open-pair cache (er_vcache) holds every open pair once: the same integer sums
    assert G.query("er_vcache_records") > 0
    G.set_option("er_bwd_fx", 1)
    G.set_option("er_vcache_use", 0)
    assert np.array_equal(gpu_backward(G, w).reshape(cfg.n_vox, cfg.nq), b)


@pytest.mark.parametrize("si", [0, 1, 2, 5])
def test_er_backward_open_pair_cache_bitwise(si):
    """Backward from the voxel-major open-pair cache (er_vcache, default) vs recomputing the pair
    geometry per call (er_vcache_use=0): the integer sums are order-free, so the bits agree; the
    cache holds exactly the pairs with an open mask cell and a non-empty energy window."""
    d = _er_desc(**ER_BWD_SHAPES[si])
    G = P.Geometry(d)
    assert 0 < G.query("er_vcache_records") <= oracle.Geometry(d).count_terms()[1]
    w = rnd(G.g_shape, 0, 170 + si)
    b1 = gpu_backward(G, w)
    G.set_option("er_vcache_use", 0)
    assert np.array_equal(gpu_backward(G, w), b1)
    G2 = P.Geometry(d, options="er_vcache=0")
    assert G2.query("er_vcache_records") == 0
    assert np.array_equal(gpu_backward(G2, w), b1)
