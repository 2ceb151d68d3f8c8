"""The fp16-rate ESAI contractions (option gemm16=1, the default; csrc/tcgemm16.cuh): W = F S~^T and
b2 = A S~ on tcgen05 kind::f16 with a two-term fp16 split of both operands (power-of-two
scales: f per row, the backward's histogram matrix from its fixed-point bound, S~ one
global).  Held to the oracle bar on the geometries, ragged shapes and hard inputs of the
other tests, and to the 3xTF32 GEMMs (option gemm16=0, which share none of this code)
at a tighter cross-check."""
import numpy as np
import pytest

import oracle
from oracle import recon
from workloads import make_config, poisson_data
from workloads.configs import seeded_rng

torch = pytest.importorskip("torch")
P = pytest.importorskip("paper_1603_06400_b200")

from test_gpu_parity import _sample, assert_parity, cuda, gpu_backward, gpu_forward, rel_l2, rnd  # noqa: E402
from test_gpu_parity_full import _log_uniform, _signed, assert_parity_signed  # noqa: E402

pytestmark = pytest.mark.gpu

OPT = "gemm16=1"


def _both(d):
    return P.Geometry(d, options=OPT), P.Geometry(d, options="gemm16=0")


@pytest.mark.parametrize("over", [
    {},
    dict(ny=5, nz=7, nq=13, det_nx=9, det_ny=23),          # one partial K chunk (nq < 32: an all-zero box)
    dict(ny=3, nz=33, nq=2, det_nx=17, det_ny=31),
    dict(ny=13, nz=23, nq=70, det_nx=37, det_ny=41),       # two K chunks, the second ragged
    dict(ny=4, nz=5, nq=16, det_nx=64, det_ny=1024, det_pitch=0.05),
    dict(q_min=0.0, q_max=0.9, nq=40),
])
def test_gemm16_small_geometries(over):
    d = make_config(0).desc()
    d.update(over)
    G, G32 = _both(d)
    O = oracle.Geometry(d)
    f, w = rnd(G.f_shape, 0, 120), rnd(G.g_shape, 0, 121)
    gf, gb = gpu_forward(G, f), gpu_backward(G, w)
    assert_parity(gf, O.forward(f), f"gemm16 {over} forward")
    assert_parity(gb, O.backward(w), f"gemm16 {over} backward")
    assert rel_l2(gf, gpu_forward(G32, f)) < 2e-6
    assert rel_l2(gb, gpu_backward(G32, w)) < 2e-6


@pytest.fixture(scope="module")
def config1():
    cfg = make_config(1)
    return cfg, P.Geometry(cfg.desc(), options=OPT), oracle.Geometry(cfg)


def test_gemm16_config1(config1):
    cfg, G, O = config1
    assert_parity(gpu_forward(G, cfg.f), O.forward(cfg.f), "gemm16 c1 forward")
    w = rnd(G.g_shape, 1, 10)
    assert_parity(gpu_backward(G, w), O.backward(w), "gemm16 c1 backward")


@pytest.mark.parametrize("kind", ["log_uniform", "signed", "row_scales"])
def test_gemm16_config1_hard_inputs(config1, kind):
    """Inputs that exercise the scales: six decades in w and f, signs, and rows of f
    whose magnitudes differ by 2^+-60 (each f row has its own power of two)."""
    cfg, G, O = config1
    if kind == "log_uniform":
        w, f = _log_uniform(G.g_shape, 1, 122), _log_uniform(G.f_shape, 1, 123)
        assert_parity(gpu_backward(G, w), O.backward(w), "gemm16 c1 backward, log-uniform w")
        assert_parity(gpu_forward(G, f), O.forward(f), "gemm16 c1 forward, log-uniform f")
    elif kind == "signed":
        w, f = _signed(G.g_shape, 1, 124), _signed(G.f_shape, 1, 125)
        assert_parity_signed(gpu_backward(G, w), O.backward(w), O.backward(np.abs(w)), "gemm16 c1 backward, signed w")
        assert_parity_signed(gpu_forward(G, f), O.forward(f), O.forward(np.abs(f)), "gemm16 c1 forward, signed f")
    else:
        f = rnd(G.f_shape, 1, 126).reshape(cfg.n_vox, cfg.nq)
        ex = seeded_rng(1, 127).integers(-60, 61, cfg.n_vox)
        f = (f * np.ldexp(1.0, ex)[:, None]).astype(np.float32).reshape(G.f_shape)
        g = gpu_forward(G, f)
        assert np.all(np.isfinite(g))
        assert_parity(g, O.forward(f), "gemm16 c1 forward, rows scaled by 2^-60 .. 2^60")
        # and the forward is linear in each row: scaling one voxel's row by 2^k scales
        # its contribution exactly (the per-row power of two absorbs it)
        f1 = np.zeros_like(f).reshape(cfg.n_vox, cfg.nq)
        f1[77] = f.reshape(cfg.n_vox, cfg.nq)[77]
        f2 = f1 * np.float32(2.0 ** 40)
        assert np.array_equal(gpu_forward(G, f2), gpu_forward(G, f1) * np.float32(2.0 ** 40))


def test_gemm16_config3_iterates():
    """Alg. 5 through cacsi_iterate (the fused forward / ratio / backward / update) with the
    fp16-rate GEMMs: b1 and three iterates against the oracle's."""
    cfg = make_config(3)
    y, r, s = poisson_data(oracle.Geometry(cfg).forward(cfg.f.astype(np.float64)), seed=3)
    d = cfg.desc()
    d["scale"] = s
    O, G = oracle.Geometry(d), P.Geometry(d, options=OPT)
    b1_ref = O.backward(np.ones(O.g_shape))
    b1 = torch.empty(G.f_shape, dtype=torch.float32, device="cuda")
    G.backward(torch.ones(G.g_shape, dtype=torch.float32, device="cuda"), b1)
    assert_parity(b1.cpu().numpy(), b1_ref, "gemm16 c3 b1")
    beta = 1e-3
    f0 = np.full(G.f_shape, (y - r).sum() / b1_ref.sum(), dtype=np.float32)
    ref_iters = recon.em_iterate(O, f0, y, r, b1_ref.astype(np.float32), beta, 3)
    f = cuda(f0)
    ws = torch.empty(G.workspace_bytes, dtype=torch.uint8, device="cuda")
    yt, rt = cuda(y), cuda(r)
    for t in range(3):
        G.iterate(f, yt, rt, b1, beta, 1, ws)
        torch.cuda.synchronize()
        assert_parity(f.cpu().numpy(), ref_iters[t], f"gemm16 c3 iterate {t + 1}")


def test_gemm16_config2_vs_tf32_and_oracle_sampled():
    cfg = make_config(2)
    G, G32 = _both(cfg.desc())
    O = oracle.Geometry(cfg)
    g16, g32 = gpu_forward(G, cfg.f), gpu_forward(G32, cfg.f)
    w = rnd(G.g_shape, 2, 10)
    b16, b32 = gpu_backward(G, w), gpu_backward(G32, w)
    assert rel_l2(g16, g32) < 2e-6 and rel_l2(b16, b32) < 2e-6
    pix = _sample(cfg.n_det, 1024, 128)
    assert_parity(g16.ravel()[pix], O.forward_pixels(cfg.f, pix), "gemm16 c2 forward, 1024 pixels")
    vox = _sample(cfg.n_vox, 128, 129)
    assert_parity(b16.reshape(cfg.n_vox, cfg.nq)[vox], O.backward_voxels(w, vox), "gemm16 c2 backward, 128 voxels")
    # deterministic
    assert np.array_equal(gpu_forward(G, cfg.f), g16) and np.array_equal(gpu_backward(G, w), b16)


@pytest.mark.parametrize("over", [{}, dict(ny=13, nz=23, nq=70, det_nx=37, det_ny=41), dict(ny=5, nz=7, nq=13)])
def test_w_tma_store_bitwise(over):
    """The W GEMM's epilogue by TMA tensor stores (w_tmast=1, the default; clipped at the
    map's edges) writes the same bits as the per-lane stores (w_tmast=0)."""
    d = make_config(1 if not over else 0).desc()
    d.update(over)
    G = P.Geometry(d, options="w_tmast=0")
    f = rnd(G.f_shape, 0, 130)
    g0 = gpu_forward(G, f)
    G.set_option("w_tmast", 1)
    assert np.array_equal(gpu_forward(G, f), g0)


@pytest.mark.parametrize("ci", [0, 1])
def test_b2_tma_store_bitwise(ci):
    """The b2 GEMM's partials by TMA tensor stores (b2_tmast=1, the default) carry the same
    bits as the per-lane stores (b2_tmast=0); empty units (tiles whose windows miss a split) store zeros either way."""
    cfg = make_config(ci)
    G = P.Geometry(cfg.desc(), options="b2_tmast=0")
    w = rnd(G.g_shape, ci, 131)
    b0 = gpu_backward(G, w)
    G.set_option("b2_tmast", 1)
    assert np.array_equal(gpu_backward(G, w), b0)


def test_b2_ring_depths_bitwise():
    """The b2 GEMM's A / B ring depths (option b2_rings) change only the pipelining."""
    cfg = make_config(1)
    G = P.Geometry(cfg.desc())
    w = rnd(G.g_shape, 1, 132)
    out = []
    for r in (0, 1, 2):
        G.set_option("b2_rings", r)
        out.append(gpu_backward(G, w))
    assert np.array_equal(out[0], out[1]) and np.array_equal(out[0], out[2])


def test_b2_tma_store_split_boundaries():
    """n_vox not a multiple of 128: the last M tile of every split overhangs into the next
    split's rows, which the 3-D tensor map clips per split (a 2-D map over [S M][nq] let
    those zero rows land in the next split's partials, a race).  Repeated, against the
    per-lane stores."""
    d = make_config(0).desc()
    d.update(ny=5, nz=7, nq=40, det_nx=9, det_ny=23)
    G = P.Geometry(d, options="b2_tmast=0")
    w = rnd(G.g_shape, 0, 133)
    ref = gpu_backward(G, w)
    G.set_option("b2_tmast", 1)
    for _ in range(30):
        assert np.array_equal(gpu_backward(G, w), ref)
