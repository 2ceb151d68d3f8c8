"""Bitwise reproducibility of the operators: the pair-cache
kernels stage data through shared memory with cp.async.bulk and mbarrier rings;
a missing proxy fence or phase error shows up as a run-to-run difference long
before it shows up as a parity failure.  The backward's sums are integers
(order-free), the forward's are fixed-order fp32 per voxel chunk, so every
repeat must be bit-identical -- and the two backward kernels (bulk-copy ring,
register-fed "flat") must agree bit for bit."""
import numpy as np
import pytest

from workloads import make_config

torch = pytest.importorskip("torch")
P = pytest.importorskip("paper_1603_06400_b200")

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("ci,q8", [(1, 0), (2, 0), (1, 2), (2, 2)])
def test_repeat_bitwise(ci, q8):
    cfg = make_config(ci)
    G = P.Geometry(cfg.desc(), options=f"pc_q8={q8}")
    f = torch.as_tensor(cfg.f).cuda()
    w = torch.as_tensor(np.random.default_rng(3).uniform(0, 1, G.g_shape).astype(np.float32)).cuda()
    g0, b0 = torch.empty(G.g_shape, device="cuda"), torch.empty(G.f_shape, device="cuda")
    G.forward(f, g0)
    G.backward(w, b0)
    reps = 12 if ci == 1 else 4
    for _ in range(reps):
        g, b = torch.empty_like(g0), torch.empty_like(b0)
        G.forward(f, g)
        G.backward(w, b)
        assert torch.equal(g, g0)
        assert torch.equal(b, b0)
    if q8 == 0:  # the register-fed flat backward reads 10-byte records
        G.set_option("pc_bwd_flat", 1)
        b = torch.empty_like(b0)
        G.backward(w, b)
        assert torch.equal(b, b0)
    G.close()


def test_cta_pair_w_gemm_bitwise():
    """The cta_group::2 W GEMM (option wgemm=1: M = 256 per CTA pair, half of
    each B chunk per SM, multicast commits) gives the same bits as the
    single-CTA A-resident GEMM (both 3xTF32: option gemm16=0)."""
    cfg = make_config(1)
    G = P.Geometry(cfg.desc(), options="gemm16=0")
    f = torch.as_tensor(cfg.f).cuda()
    out = []
    for mode in ("ar", "ar2"):
        G.set_option("wgemm", {"ar": 0, "ar2": 1}[mode])
        g = torch.empty(G.g_shape, device="cuda")
        G.forward(f, g)
        torch.cuda.synchronize()
        out.append(g)
    assert torch.equal(out[0], out[1])
    G.close()


@pytest.mark.parametrize("ci", [1, 2])
def test_pipelined_forward_bitwise(ci):
    """Option pcv_pipe=1 (software-pipelined record loads in the voxel-major forward)
    gives the same bits as the default loop."""
    cfg = make_config(ci)
    G = P.Geometry(cfg.desc())
    f = torch.as_tensor(cfg.f).cuda()
    out = []
    for mode in (0, 1):
        G.set_option("pcv_pipe", mode)
        g = torch.empty(G.g_shape, device="cuda")
        G.forward(f, g)
        torch.cuda.synchronize()
        out.append(g)
    assert torch.equal(out[0], out[1])
    G.close()


@pytest.mark.parametrize("win", [256, 512])
def test_permutation_window_bitwise(win):
    """Option pc_win (the bank-aware permutation over 256- or 512-record windows,
    segments padded to the window) moves records only within windows and adds padding
    records with P = 0: the operators give the same bits as the default."""
    cfg = make_config(1)
    # (10-byte records for both: a wider window's 128-record sub-windows may span too many
    # pixels for the 8-byte format, whose rounded tau would then differ)
    G, Gw = P.Geometry(cfg.desc(), options="pc_q8=0"), P.Geometry(cfg.desc(), options=f"pc_win={win},pc_q8=0")
    assert Gw.query("pair_cache_padded_records") >= G.query("pair_cache_padded_records")
    f = torch.as_tensor(cfg.f).cuda()
    w = torch.as_tensor(np.random.default_rng(6).uniform(0, 1, G.g_shape).astype(np.float32)).cuda()
    for H in (G, Gw):
        H.g, H.b = torch.empty(G.g_shape, device="cuda"), torch.empty(G.f_shape, device="cuda")
        H.forward(f, H.g)
        H.backward(w, H.b)
    torch.cuda.synchronize()
    assert torch.equal(G.g, Gw.g) and torch.equal(G.b, Gw.b)


def _er_medium():
    d = make_config(0, energy_resolving=1).desc()
    d.update(ny=64, nz=67, det_nx=21, det_ny=37, ne=100, nq=33,
             energy_kev=np.linspace(21.0, 149.0, 100), phi=np.linspace(1.0, 0.3, 100))
    return d


def test_er_repeat_bitwise_medium():
    """The energy-resolving operators repeated 40 times on a shape with many table chunks, 5 voxel
    splits and a ragged pixel tile: the record-fed forward's barrier-free chunk rounds (warps
    counting themselves done with a buffer, the last one refilling it; lanes running ahead once
    the next chunk has landed) and the backward's two-batch prefetch must give the same bits
    every time."""
    G = P.Geometry(_er_medium())
    assert G.query("er_fcache_records") > 0 and G.query("er_vcache_records") > 0
    rng = np.random.default_rng(5)
    f = torch.as_tensor(rng.uniform(0, 1, G.f_shape).astype(np.float32)).cuda()
    w = torch.as_tensor(rng.uniform(0, 1, G.g_shape).astype(np.float32)).cuda()
    g0, b0 = torch.empty(G.g_shape, device="cuda"), torch.empty(G.f_shape, device="cuda")
    G.forward(f, g0)
    G.backward(w, b0)
    for _ in range(40):
        g, b = torch.empty_like(g0), torch.empty_like(b0)
        G.forward(f, g)
        G.backward(w, b)
        assert torch.equal(g, g0)
        assert torch.equal(b, b0)
    G.close()


def test_er_repeat_bitwise_config4():
    """Config 4 at full size (BASELINE configs[4], the bench's launch configuration): forward and
    backward three times each, bit-identical."""
    cfg = make_config(4)
    G = P.Geometry(cfg.desc())
    assert G.query("er_fcache_records") > 0
    f = torch.as_tensor(cfg.f).cuda()
    w = torch.as_tensor(np.random.default_rng(6).uniform(0, 1, G.g_shape).astype(np.float32)).cuda()
    g0, b0 = torch.empty(G.g_shape, device="cuda"), torch.empty(G.f_shape, device="cuda")
    G.forward(f, g0)
    G.backward(w, b0)
    for _ in range(2):
        g, b = torch.empty_like(g0), torch.empty_like(b0)
        G.forward(f, g)
        G.backward(w, b)
        assert torch.equal(g, g0)
        assert torch.equal(b, b0)
    G.close()
