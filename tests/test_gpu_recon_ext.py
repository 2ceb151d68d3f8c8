"""GPU parity of the §8(f) extensions through the C ABI: the Huber penalty
(cacsi_update_ex / cacsi_iterate_ex / cacsi_neg_loglik_ex, row f4) and the
ordered-subsets path (cacsi_forward_subset / cacsi_backward_subset /
cacsi_osem, row f2) against the fp64 oracle.  Same bar as test_gpu_parity."""
import numpy as np
import pytest

import oracle
from oracle import recon
from workloads import make_config
from workloads.configs import seeded_rng

torch = pytest.importorskip("torch")
P = pytest.importorskip("paper_1603_06400_b200")

from test_gpu_parity import assert_parity, cuda  # noqa: E402

pytestmark = pytest.mark.gpu


def test_update_huber_matches_oracle():
    cfg = make_config(1)
    G = P.Geometry(cfg.desc())
    rng = np.random.default_rng(31)
    f_hat = rng.uniform(0.05, 2.0, G.f_shape).astype(np.float32)
    b1 = rng.uniform(0.5, 3.0, G.f_shape).astype(np.float32)
    b2 = rng.uniform(0.1, 3.0, G.f_shape).astype(np.float32)
    out = torch.empty(G.f_shape, dtype=torch.float32, device="cuda")
    for delta in (0.02, 0.3, 10.0):
        for beta in (0.0, 1e-3, 0.5):
            G.update_ex(cuda(f_hat), cuda(b1), cuda(b2), beta, ("huber", delta), out)
            torch.cuda.synchronize()
            ref = recon.update(f_hat, b1, b2, beta, recon.Penalty("huber", delta))
            assert_parity(out.cpu().numpy(), ref, f"update huber d={delta} b={beta}", l2=1e-6, mr=1e-5)
    # quadratic through the _ex entry point == the plain cacsi_update
    q = torch.empty_like(out)
    G.update_ex(cuda(f_hat), cuda(b1), cuda(b2), 1e-3, None, out)
    G.update(cuda(f_hat), cuda(b1), cuda(b2), 1e-3, q)
    torch.cuda.synchronize()
    assert torch.equal(out, q)
    G.close()


def test_invalid_penalty_rejected():
    cfg = make_config(0)
    G = P.Geometry(cfg.desc())
    x = torch.ones(G.f_shape, dtype=torch.float32, device="cuda")
    for pen in (P.binding.Penalty(1, 0.0), P.binding.Penalty(1, -1.0), P.binding.Penalty(7, 1.0)):
        with pytest.raises(P.CacsiError) as ei:
            G.update_ex(x, x, x, 1e-3, pen, torch.empty_like(x))
        assert ei.value.status == P.binding.CACSI_ERR_INVALID
    G.close()


@pytest.fixture(scope="module")
def em0():
    """Config-0 Poisson problem (the oracle pins' EM setup)."""
    cfg = make_config(0)
    O = oracle.Geometry(cfg)
    f_true = cfg.f.astype(np.float64)
    s = 50.0 / O.forward(f_true).mean()
    d = cfg.desc()
    d["scale"] = s
    O = oracle.Geometry(d)
    G = P.Geometry(d)
    y = seeded_rng(0, 8).poisson(O.forward(f_true) + 1.0).astype(np.float32)
    r = np.ones(O.g_shape, np.float32)
    return cfg, O, G, y, r


def test_iterate_and_objective_huber(em0):
    cfg, O, G, y, r = em0
    pen = recon.Penalty("huber", 0.05)
    beta = 2e-2
    b1_ref = O.backward(np.ones(O.g_shape))
    b1 = torch.empty(G.f_shape, dtype=torch.float32, device="cuda")
    G.backward(torch.ones(G.g_shape, dtype=torch.float32, device="cuda"), b1)
    f0 = np.full(G.f_shape, (y - r).sum() / b1_ref.sum(), dtype=np.float32)
    ref = recon.em_iterate(O, f0, y, r, b1.cpu().numpy(), beta, 3, pen=pen)
    f = cuda(f0)
    ws = torch.empty(G.workspace_bytes, dtype=torch.uint8, device="cuda")
    for t in range(3):
        G.iterate_ex(f, cuda(y), cuda(r), b1, beta, ("huber", 0.05), 1, ws)
        torch.cuda.synchronize()
        assert_parity(f.cpu().numpy(), ref[t], f"huber iterate {t + 1}")  # each iterate at the operators' bar
    fx = cfg.f.astype(np.float32)
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    G.neg_loglik_ex(cuda(fx), cuda(y), cuda(r), beta, ("huber", 0.05), out, ws)
    assert out.item() == pytest.approx(recon.objective(O.forward(fx), y, r, fx, beta, pen), rel=1e-6)


def _subset_lists(cfg, rho_x, rho_y):
    sub = P.binding.symmetric_subsets(cfg.det_nx, cfg.det_ny, rho_x, rho_y).ravel()
    nsub = int(sub.max()) + 1
    lists = [np.flatnonzero(sub == p).astype(np.int32) for p in range(nsub)]
    return sub, lists


@pytest.mark.parametrize("ci,er,algo", [(0, 0, None), (1, 0, None), (0, 1, None), (0, 0, "direct")])
def test_subset_operators(ci, er, algo):
    """A_p f = (A f)|_p (zeros elsewhere) and A_p^T w = A^T (w 1_p), for ESAI
    handles (listed pairs only) and the restricted full operator of the
    energy-resolving / direct handles; subsets sum to the full operators."""
    cfg = make_config(ci, energy_resolving=er)
    O = oracle.Geometry(cfg)
    G = P.Geometry(cfg.desc(), options="direct=1" if algo == "direct" else None)
    rx, ry = (4, 8) if ci == 0 else (8, 16)
    sub, lists = _subset_lists(cfg, rx, ry)
    f = cfg.f
    w = seeded_rng(40 + ci, 1).uniform(0.5, 1.5, O.g_shape).astype(np.float32)
    g = torch.empty(G.g_shape, dtype=torch.float32, device="cuda")
    b = torch.empty(G.f_shape, dtype=torch.float32, device="cuda")
    gsum = np.zeros(O.g_shape)
    for p in (0, len(lists) // 2, len(lists) - 1):
        pix = lists[p]
        G.forward_subset(cuda(f), torch.as_tensor(pix).cuda(), g)
        G.backward_subset(cuda(w), torch.as_tensor(pix).cuda(), b)
        torch.cuda.synchronize()
        gr = np.zeros(O.g_shape).reshape(cfg.n_det, -1)
        gr[pix] = O.forward_pixels(f, pix).reshape(len(pix), -1)
        gr = gr.reshape(O.g_shape)
        assert_parity(g.cpu().numpy(), gr, f"c{ci} er{er} {algo} forward subset {p}")
        assert not np.any(g.cpu().numpy().reshape(cfg.n_det, -1)[sub != p])
        assert_parity(b.cpu().numpy(), O.backward_pixels(w, pix), f"c{ci} er{er} {algo} backward subset {p}")
    if ci == 0:
        for pix in lists:
            G.forward_subset(cuda(f), torch.as_tensor(pix).cuda(), g)
            torch.cuda.synchronize()
            gsum += g.cpu().numpy()
        # the subset forwards compute each pair's P exactly (on the fly); the full forward
        # of a default handle reads it rounded to 28 bits from the 8-byte pair cache
        # (reading R23), so the tight sum check runs against the 10-byte cache
        full = torch.empty_like(g)
        Gf = P.Geometry(cfg.desc(), options="direct=1" if algo == "direct" else "pc_q8=0")
        Gf.forward(cuda(f), full)
        torch.cuda.synchronize()
        Gf.close()
        assert_parity(gsum, full.cpu().numpy(), "sum of subset forwards", l2=1e-6, mr=1e-5)
    G.close()


def _osem_setup(O, G, cfg, lists):
    b1s = torch.empty((len(lists),) + G.f_shape, dtype=torch.float32, device="cuda")
    ones = torch.ones(G.g_shape, dtype=torch.float32, device="cuda")
    for p, pix in enumerate(lists):
        G.backward_subset(ones, torch.as_tensor(pix).cuda(), b1s[p])
    offs = np.concatenate([[0], np.cumsum([len(x) for x in lists])]).astype(np.int32)
    allpix = torch.as_tensor(np.concatenate(lists)).cuda()
    return b1s, allpix, offs


def test_osem_config0(em0):
    """Alg. 6 with the 16-subset symmetric partition: two outer iterations
    (32 sub-iterations) through cacsi_osem vs the oracle's osem_iterate."""
    cfg, O, G, y, r = em0
    sub, lists = _subset_lists(cfg, 4, 8)
    b1s, allpix, offs = _osem_setup(O, G, cfg, lists)
    b1_ref = O.backward(np.ones(O.g_shape))
    f0 = np.full(G.f_shape, (y - r).sum() / b1_ref.sum(), dtype=np.float32)
    beta = 1e-3
    for pen, tag in ((None, "quadratic"), (("huber", 0.05), "huber")):
        rp = recon.Penalty("huber", 0.05) if pen else recon.QUADRATIC
        ref = recon.osem_iterate(O, f0, y, r, sub.reshape(O.g_shape), beta, 2, pen=rp, restricted=True)
        f = cuda(f0)
        ws = torch.empty(G.workspace_bytes, dtype=torch.uint8, device="cuda")
        for t in range(2):
            G.osem(f, cuda(y), cuda(r), b1s, allpix, offs, beta, pen, 1, ws)
            torch.cuda.synchronize()
            assert_parity(f.cpu().numpy(), ref[t], f"osem {tag} outer {t + 1}", l2=1e-5 * (t + 1),
                          mr=1e-4 * (t + 1))


@pytest.fixture(scope="module")
def osem3():
    cfg = make_config(1)
    O = oracle.Geometry(cfg)
    lt = O.forward(cfg.f.astype(np.float64))
    s = 1e4 / lt.mean()
    d = cfg.desc()
    d["scale"] = s
    O = oracle.Geometry(d)
    G = P.Geometry(d)
    y = seeded_rng(3, 2).poisson(s * lt + 5.0).astype(np.float32)
    r = np.full(O.g_shape, 5.0, np.float32)
    sub, lists = _subset_lists(cfg, 8, 16)
    assert len(lists) == 64  # the paper's 64 subsets
    b1s, allpix, offs = _osem_setup(O, G, cfg, lists)
    b1_ref = O.backward(np.ones(O.g_shape))
    f0 = np.full(G.f_shape, (y - r).sum() / b1_ref.sum(), dtype=np.float32)
    return cfg, O, G, y, r, sub, lists, b1s, allpix, offs, f0


def test_osem_config3_one_subiteration(osem3):
    """One sub-iteration of Alg. 6 (subset p alone, penalty weight beta / 64)
    from the same f: parity on the voxels the subset sees (b1_p >= 1e-3 of its
    max; a barely-seen voxel's update b2_p / b1_p divides two tiny sums)."""
    cfg, O, G, y, r, sub, lists, b1s, allpix, offs, f0 = osem3
    ws = torch.empty(G.workspace_bytes, dtype=torch.uint8, device="cuda")
    beta = 1e-3
    for p in (0, 31, 63):
        pix = lists[p]
        f = cuda(f0)
        G.osem(f, cuda(y), cuda(r), b1s[p:p + 1].contiguous(), torch.as_tensor(pix).cuda(), [0, len(pix)],
               beta / 64, None, 1, ws)
        torch.cuda.synchronize()
        b1r = O.backward_pixels(np.ones(O.g_shape), pix)
        gr = np.zeros(cfg.n_det)
        gr[pix] = O.forward_pixels(f0, pix)
        ind = (sub == p).reshape(O.g_shape)
        rat = recon.ratio(gr.reshape(O.g_shape), y, r) * ind
        ref = recon.update(f0, b1r, O.backward_pixels(rat, pix), beta / 64)
        seen = b1r >= 1e-3 * b1r.max()
        assert_parity(f.cpu().numpy()[seen], ref[seen], f"osem c3 sub-iteration {p}")


def test_osem_config3_outer_iteration(osem3):
    """One outer iteration (64 sub-iterations) through cacsi_osem vs the
    oracle's osem_iterate, at the operators' bar (the subset backward's
    fixed-point unit is set by the subset's own weights, k_absmax)."""
    cfg, O, G, y, r, sub, lists, b1s, allpix, offs, f0 = osem3
    beta = 1e-3
    ref = recon.osem_iterate(O, f0, y, r, sub.reshape(O.g_shape), beta, 1, restricted=True)
    f = cuda(f0)
    ws = torch.empty(G.workspace_bytes, dtype=torch.uint8, device="cuda")
    G.osem(f, cuda(y), cuda(r), b1s, allpix, offs, beta, None, 1, ws)
    torch.cuda.synchronize()
    assert_parity(f.cpu().numpy(), ref[0], "osem c3 64 subsets outer 1")
