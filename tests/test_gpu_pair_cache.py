"""The pair cache: both operators with and without it
(CACSI_PAIR_CACHE=0) against the oracle, its record count against the
oracle's exact count of open pairs, and the two paths against each other."""
import json
import math
import os

import numpy as np
import pytest

import oracle
from workloads import make_config

torch = pytest.importorskip("torch")
P = pytest.importorskip("paper_1603_06400_b200")

from test_gpu_parity import _sample, assert_parity, gpu_backward, gpu_forward, rnd  # noqa: E402

pytestmark = pytest.mark.gpu
COUNTS = json.load(open(os.path.join(os.path.dirname(os.path.dirname(__file__)), "workloads", "work_counts.json")))


def handles(d):
    Gc = P.Geometry(d)
    Gn = P.Geometry(d, options="pair_cache=0")
    return Gc, Gn


@pytest.mark.parametrize("ci", [1, 2])
def test_record_count_is_the_open_pair_count(ci):
    cfg = make_config(ci)
    Gc, Gn = handles(cfg.desc())
    assert Gc.query("pair_cache_records") == COUNTS[str(cfg.seed)]["open_pairs"]
    assert Gn.query("pair_cache_records") == 0
    assert Gc.query("pair_cache_tau_bits") >= 16
    # default (pc_q8=2): P rounded to 28 bits + (b, tau): 8 B per record, and 2 B of pixel base
    # per 128-record window (the pixel's offset from it rides in P's low nibble and 5 b-word bits)
    assert Gc.query("pair_cache_record_bytes") == 8
    assert Gc.query("pair_cache_window_base_bytes") == 2 * Gc.query("pair_cache_padded_records") // 128
    # pc_q8=0: P (4 B) + packed (b, tau) (4 B) + pixel q (2 B for n_det <= 65536)
    G10 = P.Geometry(cfg.desc(), options="pc_q8=0")
    assert G10.query("pair_cache_record_bytes") == 8 + (2 if cfg.n_det <= 65536 else 4)
    assert G10.query("pair_cache_window_base_bytes") == 0
    G10.close()
    Gc.close()
    Gn.close()


def test_cache_on_off_config1():
    cfg = make_config(1)
    O = oracle.Geometry(cfg)
    Gc, Gn = handles(cfg.desc())
    gr = O.forward(cfg.f)
    w = rnd(Gc.g_shape, 1, 70)
    br = O.backward(w)
    for tag, G in (("cache", Gc), ("on-the-fly", Gn)):
        assert_parity(gpu_forward(G, cfg.f), gr, f"c1 {tag} forward")
        assert_parity(gpu_backward(G, w), br, f"c1 {tag} backward")
    assert_parity(gpu_forward(Gc, cfg.f), gpu_forward(Gn, cfg.f), "c1 cache vs on-the-fly forward", l2=1e-6, mr=1e-5)
    Gc.close()
    Gn.close()


def test_on_the_fly_config2_sampled():
    """Full-size config 2 on the kernels that recompute the pair geometry per
    call (the subset operators and the no-cache fallback use them)."""
    cfg = make_config(2)
    O = oracle.Geometry(cfg)
    G = P.Geometry(cfg.desc(), options="pair_cache=0")
    g = gpu_forward(G, cfg.f).ravel()
    pix = _sample(cfg.n_det, 96, 11)
    assert_parity(g[pix], O.forward_pixels(cfg.f, pix), "c2 on-the-fly forward sampled")
    w = rnd(G.g_shape, 2, 71)
    b = gpu_backward(G, w).reshape(cfg.n_vox, cfg.nq)
    vox = _sample(cfg.n_vox, 12, 12)
    assert_parity(b[vox], O.backward_voxels(w, vox), "c2 on-the-fly backward sampled")
    G.close()


def test_sai_without_cache():
    cfg = make_config(1)
    d = cfg.desc()
    d.update(sai_n_theta=250, sai_theta_min=0.2 * math.pi / 180, sai_theta_max=math.pi / 6)
    G, O = P.Geometry(d, options="pair_cache=0"), oracle.Geometry(d)
    assert_parity(gpu_forward(G, cfg.f), O.forward(cfg.f), "c1 SAI on-the-fly forward")
    w = rnd(G.g_shape, 1, 72)
    assert_parity(gpu_backward(G, w), O.backward(w), "c1 SAI on-the-fly backward")
    G.close()


def test_per_list_forward_config1():
    """The per-list pair-cache forward (used when the voxel-major kernel's
    shared-memory window does not fit; option pc_fwd_list=1 forces it) against
    the oracle and against the voxel-major kernel."""
    cfg = make_config(1)
    O = oracle.Geometry(cfg)
    G = P.Geometry(cfg.desc(), options="pc_q8=0")  # the same 10-byte records as the plain layout
    assert G.query("pair_cache_records") > 0
    gv = gpu_forward(G, cfg.f)
    # the per-list kernel needs the plain (list-ordered, unpadded) layout
    Gp = P.Geometry(cfg.desc(), options="pc_plain=1")
    assert Gp.query("pair_cache_padded_records") == Gp.query("pair_cache_records")
    Gp.set_option("pc_fwd_list", 1)
    gl = gpu_forward(Gp, cfg.f)
    G.set_option("pc_fwd_list", 1)
    assert torch.equal(torch.as_tensor(gpu_forward(G, cfg.f)), torch.as_tensor(gv))  # ignored by a bank-ordered cache
    assert_parity(gl, O.forward(cfg.f), "c1 per-list cache forward")
    assert_parity(gl, gv, "c1 per-list vs voxel-major forward", l2=1e-6, mr=1e-5)
    w = rnd(G.g_shape, 1, 73)
    bp, bo = gpu_backward(Gp, w), gpu_backward(G, w)
    assert np.array_equal(np.asarray(bp), np.asarray(bo))  # integer sums: the record order is irrelevant
    G.close()
    Gp.close()


def test_wide_detector_uint32_pixels():
    """n_det > 65536: the pair cache stores the pixel as uint32 (12-byte records)
    and both pair-cache kernels take their uint32 instantiation."""
    cfg = make_config(0)
    d = cfg.desc()
    d.update(ny=4, nz=3, nq=8, det_nx=260, det_ny=256, det_pitch=0.1)
    G, O = P.Geometry(d), oracle.Geometry(d)
    assert G.n_det > 65536
    assert G.query("pair_cache_records") > 0
    assert G.query("pair_cache_record_bytes") == 12
    f, w = rnd(G.f_shape, 0, 80), rnd(G.g_shape, 0, 81)
    assert_parity(gpu_forward(G, f), O.forward(f), "wide detector forward")
    assert_parity(gpu_backward(G, w), O.backward(w), "wide detector backward")
    G.close()


@pytest.mark.parametrize("ci", [1, 2])
def test_forward_recomputed_P_matches_stored(ci):
    """Option pc_fwd_geom=1: the voxel-major forward recomputes each record's P from the
    pixel index and the voxel (6-byte records, translation-symmetric s_y) instead of
    reading it; same operator up to fp32 rounding of P, and the oracle bar (config 1).
    (10-byte records: the recomputing variant reads b, tau and the pixel from them.)"""
    cfg = make_config(ci)
    G = P.Geometry(cfg.desc(), options="pc_q8=0")
    g0 = gpu_forward(G, cfg.f)
    G.set_option("pc_fwd_geom", 1)
    g1 = gpu_forward(G, cfg.f)
    assert_parity(g1, g0, f"c{ci} recomputed-P vs stored-P forward", l2=1e-6, mr=1e-5)
    if ci == 1:
        assert_parity(g1, oracle.Geometry(cfg).forward(cfg.f), "c1 recomputed-P forward")
    G.close()



@pytest.mark.parametrize("ci,mode", [(1, 1), (2, 1), (1, 2), (2, 2)])
def test_8_byte_records_match_10_byte(ci, mode):
    """The packed 8-byte records against the 10-byte format and, on config 1, the oracle.
    Mode 1 rounds tau to tbits - 9 bits (10 on config 2: each interpolation weight moves by up
    to 2^-11), so the formats agree at the oracle bar, not bit for bit; mode 2 keeps tbits - 5
    tau bits and rounds P to 28 bits (relative error <= 2^-20 per pair) and is held to the
    10-byte format ten times tighter (reading R23)."""
    cfg = make_config(ci)
    G8, G10 = P.Geometry(cfg.desc(), options=f"pc_q8={mode}"), P.Geometry(cfg.desc(), options="pc_q8=0")
    assert G8.query("pair_cache_record_bytes") == 8 and G10.query("pair_cache_record_bytes") == 10
    w = rnd(G8.g_shape, ci, 74)
    l2, mr = (1e-5, 1e-4) if mode == 1 else (1e-6, 1e-5)
    assert_parity(gpu_forward(G8, cfg.f), gpu_forward(G10, cfg.f), f"c{ci} 8-byte ({mode}) vs 10-byte forward", l2, mr)
    assert_parity(gpu_backward(G8, w), gpu_backward(G10, w), f"c{ci} 8-byte ({mode}) vs 10-byte backward", l2, mr)
    if ci == 1:
        O = oracle.Geometry(cfg)
        assert_parity(gpu_forward(G8, cfg.f), O.forward(cfg.f), f"c1 8-byte ({mode}) forward")
        assert_parity(gpu_backward(G8, w), O.backward(w), f"c1 8-byte ({mode}) backward")
    G8.close()
    G10.close()


@pytest.mark.parametrize("ci", [1, 2])
def test_padding_pixels_closed_bitwise(ci):
    """Padding records carry a pixel that is closed for their voxel (k_pc_fill), so the
    voxel-major forward adds their zero in place (pcv_padq=1, the default) -- the same
    bits as redirecting them to the dummy slots (pcv_padq=0)."""
    cfg = make_config(ci)
    G = P.Geometry(cfg.desc())
    assert G.query("pair_cache_padding_closed") == 1
    f = torch.as_tensor(cfg.f).cuda()
    out = []
    for v in (1, 0):
        G.set_option("pcv_padq", v)
        g = torch.empty(G.g_shape, device="cuda")
        G.forward(f, g)
        torch.cuda.synchronize()
        out.append(g)
    assert torch.equal(out[0], out[1])


@pytest.mark.parametrize("ci", [1, 2])
def test_backward_l1_prefetch_bitwise(ci):
    """The ring backward's L1 prefetch of the next chunk's w lines (pcb_pfl1=1, the default)
    changes no arithmetic: the same bits as without it."""
    cfg = make_config(ci)
    G = P.Geometry(cfg.desc())
    w = rnd(G.g_shape, ci, 76)
    b1 = gpu_backward(G, w)
    G.set_option("pcb_pfl1", 0)
    assert np.array_equal(gpu_backward(G, w), b1)


@pytest.mark.parametrize("ci", [1, 2])
def test_lane_permutation_bitwise(ci):
    """The bank-aware permutation with one window per lane (k_pc_perm128, pc_perm_lane=1, the
    default) makes the same assignment as the warp-per-window greedy (pc_perm_lane=0): the
    operators give the same bits."""
    cfg = make_config(ci)
    f = rnd(cfg.f_shape, ci, 77)
    w = rnd((cfg.det_nx, cfg.det_ny), ci, 78)
    res = []
    for v in (1, 0):
        G = P.Geometry(cfg.desc(), options=f"pc_perm_lane={v}")
        res.append((gpu_forward(G, f), gpu_backward(G, w)))
        G.close()
    assert np.array_equal(res[0][0], res[1][0])
    assert np.array_equal(res[0][1], res[1][1])
