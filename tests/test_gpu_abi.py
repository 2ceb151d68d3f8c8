"""GPU-side ABI behaviour: error codes of the §8(f) entry points, empty and
degenerate subsets, determinism, host/device agreement and concurrent calls
on one handle from two streams (include/cacsi.h conventions)."""
import math

import numpy as np
import pytest

import oracle
from workloads import make_config

torch = pytest.importorskip("torch")
P = pytest.importorskip("paper_1603_06400_b200")

from test_gpu_parity import assert_parity, cuda, gpu_backward, gpu_forward, rnd  # noqa: E402

pytestmark = pytest.mark.gpu
B = P.binding


def _status(fn):
    try:
        fn()
    except P.CacsiError as e:
        return e.status
    return B.CACSI_OK


def test_subset_argument_errors():
    cfg = make_config(0)
    G = P.Geometry(cfg.desc())
    f = cuda(cfg.f)
    g = torch.empty(G.g_shape, dtype=torch.float32, device="cuda")
    too_many = torch.arange(cfg.n_det + 1, dtype=torch.int32, device="cuda")
    assert _status(lambda: G.forward_subset(f, too_many, g)) == B.CACSI_ERR_INVALID
    # NULL pixel list with a positive count
    st = B.lib().cacsi_forward_subset(G.handle, f.data_ptr(), None, 3, g.data_ptr(), None)
    assert st == B.CACSI_ERR_NULL
    # empty subset: zero output
    g.fill_(7.0)
    G.forward_subset(f, torch.empty(0, dtype=torch.int32, device="cuda"), g)
    b = torch.full(G.f_shape, 7.0, dtype=torch.float32, device="cuda")
    G.backward_subset(cuda(np.ones(G.g_shape)), torch.empty(0, dtype=torch.int32, device="cuda"), b)
    torch.cuda.synchronize()
    assert not g.any() and not b.any()
    G.close()


def test_osem_argument_errors():
    cfg = make_config(0)
    G = P.Geometry(cfg.desc())
    f = cuda(np.ones(G.f_shape))
    y = cuda(np.ones(G.g_shape))
    ws = torch.empty(G.workspace_bytes, dtype=torch.uint8, device="cuda")
    pix = torch.arange(cfg.n_det, dtype=torch.int32, device="cuda")
    b1 = cuda(np.ones((2,) + G.f_shape))
    for offs in ([1, 128, 256], [0, 200, 100], [0, 128, 300]):
        assert _status(lambda: G.osem(f, y, y, b1, pix, offs, 1e-3, None, 1, ws)) == B.CACSI_ERR_INVALID
    assert _status(lambda: G.osem(f, y, y, b1, pix, [0, 128, 256], -1.0, None, 1, ws)) == B.CACSI_ERR_INVALID
    assert _status(lambda: G.osem(f, y, y, b1, pix, [0, 128, 256], 1e-3, ("huber", 0.0), 1, ws)) == \
        B.CACSI_ERR_INVALID
    G.osem(f, y, y, b1, pix, [0, 128, 256], 1e-3, None, 0, ws)  # zero iterations: ok, f untouched
    torch.cuda.synchronize()
    assert torch.equal(f, cuda(np.ones(G.f_shape)))
    G.close()


def test_subset_operators_deterministic():
    cfg = make_config(1)
    G = P.Geometry(cfg.desc())
    sub = B.symmetric_subsets(cfg.det_nx, cfg.det_ny, 8, 16).ravel()
    pix = torch.as_tensor(np.flatnonzero(sub == 5).astype(np.int32)).cuda()
    w = cuda(rnd(G.g_shape, 1, 60))
    b1 = torch.empty(G.f_shape, dtype=torch.float32, device="cuda")
    b2 = torch.empty_like(b1)
    G.backward_subset(w, pix, b1)
    G.backward_subset(w, pix, b2)
    f = cuda(cfg.f)
    g1 = torch.empty(G.g_shape, dtype=torch.float32, device="cuda")
    g2 = torch.empty_like(g1)
    G.forward_subset(f, pix, g1)
    G.forward_subset(f, pix, g2)
    torch.cuda.synchronize()
    assert torch.equal(b1, b2) and torch.equal(g1, g2)
    G.close()


def test_sai_subset_operators():
    """Subset operators of a scatter-angle-interpolation handle against the SAI
    oracle restricted to the subset."""
    cfg = make_config(1)
    d = cfg.desc()
    d.update(sai_n_theta=250, sai_theta_min=0.2 * math.pi / 180, sai_theta_max=math.pi / 6)
    G, O = P.Geometry(d), oracle.Geometry(d)
    sub = B.symmetric_subsets(cfg.det_nx, cfg.det_ny, 8, 16).ravel()
    pixn = np.flatnonzero(sub == 9).astype(np.int32)
    pix = torch.as_tensor(pixn).cuda()
    g = torch.empty(G.g_shape, dtype=torch.float32, device="cuda")
    G.forward_subset(cuda(cfg.f), pix, g)
    w = rnd(G.g_shape, 1, 61)
    b = torch.empty(G.f_shape, dtype=torch.float32, device="cuda")
    G.backward_subset(cuda(w), pix, b)
    torch.cuda.synchronize()
    assert_parity(g.cpu().numpy().ravel()[pixn], O.forward_pixels(cfg.f, pixn), "SAI forward subset")
    assert_parity(b.cpu().numpy(), O.backward_pixels(w, pixn), "SAI backward subset")
    G.close()


def test_two_streams_one_handle():
    """Calls on one handle from two streams (internal scratch is stream-ordered,
    include/cacsi.h) give the same results as sequential calls."""
    cfg = make_config(1)
    G = P.Geometry(cfg.desc())
    f1, f2 = cuda(cfg.f), cuda(rnd(G.f_shape, 1, 62))
    w1, w2 = cuda(rnd(G.g_shape, 1, 63)), cuda(rnd(G.g_shape, 1, 64))
    ref = [gpu_forward(G, f1.cpu().numpy()), gpu_forward(G, f2.cpu().numpy()),
           gpu_backward(G, w1.cpu().numpy()), gpu_backward(G, w2.cpu().numpy())]
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    g1 = torch.empty(G.g_shape, dtype=torch.float32, device="cuda")
    g2 = torch.empty_like(g1)
    b1 = torch.empty(G.f_shape, dtype=torch.float32, device="cuda")
    b2 = torch.empty_like(b1)
    torch.cuda.synchronize()
    for _ in range(3):
        with torch.cuda.stream(s1):
            G.forward(f1, g1)
            G.backward(w1, b1)
        with torch.cuda.stream(s2):
            G.forward(f2, g2)
            G.backward(w2, b2)
    torch.cuda.synchronize()
    for got, want in zip((g1, g2, b1, b2), ref):
        np.testing.assert_array_equal(got.cpu().numpy(), want)
    G.close()


@pytest.mark.parametrize("n_iter", [0, 1, 3])
def test_iterate_host_matches_device_iterate(n_iter):
    """cacsi_iterate_host (inputs from host buffers; y, r, b1 uploaded on a side
    stream while the forward runs, ping-pong iterates) gives bit-identical
    iterates to cacsi_iterate on device buffers."""
    cfg = make_config(1)
    G = P.Geometry(cfg.desc())
    rng = np.random.default_rng(11)
    f0 = rng.uniform(0.5, 1.5, G.f_shape).astype(np.float32)
    y = rng.poisson(50.0, G.g_shape).astype(np.float32)
    r = np.full(G.g_shape, 2.0, dtype=np.float32)
    b1 = rng.uniform(1.0, 2.0, G.f_shape).astype(np.float32)
    fh = torch.as_tensor(f0.copy()).pin_memory()
    G.iterate_host(fh, torch.as_tensor(y).pin_memory(), torch.as_tensor(r).pin_memory(),
                   torch.as_tensor(b1).pin_memory(), 1e-3, n_iter)
    fd = torch.as_tensor(f0).cuda()
    ws = torch.empty(G.workspace_bytes, dtype=torch.uint8, device="cuda")
    G.iterate(fd, torch.as_tensor(y).cuda(), torch.as_tensor(r).cuda(), torch.as_tensor(b1).cuda(), 1e-3, n_iter, ws)
    torch.cuda.synchronize()
    assert np.array_equal(fh.numpy(), fd.cpu().numpy())
    G.close()


@pytest.mark.parametrize("ci,delta", [(1, 0.0), (1, 0.05), (2, 0.0)])
def test_fused_iterate_matches_operator_sequence(ci, delta):
    """cacsi_iterate on an ESAI handle fuses the ratio (and max |w|) into the
    forward's final partial sum and the update into the backward's: the iterate
    is bit-identical to calling cacsi_forward, cacsi_ratio, cacsi_backward and
    cacsi_update in turn (two iterations: the ping-pong buffers are exercised)."""
    cfg = make_config(ci)
    G = P.Geometry(cfg.desc())
    rng = np.random.default_rng(21)
    f0 = rng.uniform(0.5, 1.5, G.f_shape).astype(np.float32)
    y = torch.as_tensor(rng.poisson(50.0, G.g_shape).astype(np.float32)).cuda()
    r = torch.full(G.g_shape, 2.0, device="cuda")
    b1 = torch.as_tensor(rng.uniform(1.0, 2.0, G.f_shape).astype(np.float32)).cuda()
    beta = 1e-3
    pen = ("huber", delta) if delta > 0.0 else ("quadratic", 0.0)
    fd = torch.as_tensor(f0).cuda()
    ws = torch.empty(G.workspace_bytes, dtype=torch.uint8, device="cuda")
    G.iterate_ex(fd, y, r, b1, beta, pen, 2, ws)
    fs = torch.as_tensor(f0).cuda()
    l = torch.empty(G.g_shape, device="cuda")
    b2 = torch.empty(G.f_shape, device="cuda")
    fn = torch.empty(G.f_shape, device="cuda")
    for _ in range(2):
        G.forward(fs, l)
        G.ratio(l, y, r, l)
        G.backward(l, b2)
        G.update_ex(fs, b1, b2, beta, pen, fn)
        fs.copy_(fn)
    torch.cuda.synchronize()
    assert torch.equal(fd, fs)
    G.close()


@pytest.mark.parametrize("n_iter", [1, 2])
def test_iterate_host_ragged_chunks(n_iter):
    """Ragged geometry (299 voxels = 3 M tiles: the four f upload chunks are 128, 128,
    43 and 0 rows; nq = 70: a 3-chunk A panel): cacsi_iterate_host, cacsi_iterate
    and the operator sequence give the same bits."""
    cfg = make_config(0, ny=13, nz=23, nq=70, det_nx=37, det_ny=41)
    G = P.Geometry(cfg.desc())
    rng = np.random.default_rng(5)
    f0 = rng.uniform(0.5, 1.5, G.f_shape).astype(np.float32)
    y = rng.poisson(20.0, G.g_shape).astype(np.float32)
    r = np.full(G.g_shape, 1.0, dtype=np.float32)
    b1 = rng.uniform(1.0, 2.0, G.f_shape).astype(np.float32)
    fh = torch.as_tensor(f0.copy()).pin_memory()
    G.iterate_host(fh, torch.as_tensor(y).pin_memory(), torch.as_tensor(r).pin_memory(),
                   torch.as_tensor(b1).pin_memory(), 1e-3, n_iter)
    yd, rd, b1d = (torch.as_tensor(a).cuda() for a in (y, r, b1))
    fd = torch.as_tensor(f0).cuda()
    ws = torch.empty(G.workspace_bytes, dtype=torch.uint8, device="cuda")
    G.iterate(fd, yd, rd, b1d, 1e-3, n_iter, ws)
    fs = torch.as_tensor(f0).cuda()
    l = torch.empty(G.g_shape, device="cuda")
    b2 = torch.empty(G.f_shape, device="cuda")
    fn = torch.empty(G.f_shape, device="cuda")
    for _ in range(n_iter):
        G.forward(fs, l)
        G.ratio(l, yd, rd, l)
        G.backward(l, b2)
        G.update(fs, b1d, b2, 1e-3, fn)
        fs.copy_(fn)
    torch.cuda.synchronize()
    assert np.array_equal(fh.numpy(), fd.cpu().numpy())
    assert torch.equal(fd, fs)
    G.close()


def test_subset_backward_list_matches_mask():
    """The list-driven subset backward (warp per voxel over the listed pixels)
    and the bitmap-masked one deposit the same integers: bit-identical."""
    cfg = make_config(1)
    G = P.Geometry(cfg.desc())
    sub = P.binding.symmetric_subsets(cfg.det_nx, cfg.det_ny, 8, 16).ravel()
    w = torch.as_tensor(np.random.default_rng(9).uniform(0, 1, G.g_shape).astype(np.float32)).cuda()
    for p in (0, 5, 63):
        px = torch.as_tensor(np.flatnonzero(sub == p).astype(np.int32)).cuda()
        out = []
        for mode in ("list", "mask"):
            G.set_option("subset_bwd_mask", int(mode == "mask"))
            b = torch.empty(G.f_shape, device="cuda")
            G.backward_subset(w, px, b)
            torch.cuda.synchronize()
            out.append(b)
        assert torch.equal(out[0], out[1])
    G.close()


def test_osem_graph_replay_matches_stream_launches():
    """cacsi_osem replays a captured CUDA graph of the outer iteration (cached per
    handle while the arguments match); the iterates are bit-identical to plain
    stream launches (option graphs=0), including after the arguments change."""
    cfg = make_config(0)
    G = P.Geometry(cfg.desc())
    sub = P.binding.symmetric_subsets(cfg.det_nx, cfg.det_ny, 2, 4).ravel()
    nsub = int(sub.max()) + 1
    lists = [np.flatnonzero(sub == p).astype(np.int32) for p in range(nsub)]
    offs = np.concatenate([[0], np.cumsum([len(x) for x in lists])]).astype(np.int32)
    allpix = torch.as_tensor(np.concatenate(lists)).cuda()
    ones = torch.ones(G.g_shape, device="cuda")
    b1s = torch.empty((nsub,) + G.f_shape, device="cuda")
    for p in range(nsub):
        G.backward_subset(ones, allpix[offs[p]:offs[p + 1]], b1s[p])
    rng = np.random.default_rng(4)
    y = torch.as_tensor(rng.poisson(50.0, G.g_shape).astype(np.float32)).cuda()
    r = torch.full(G.g_shape, 2.0, device="cuda")
    ws = torch.empty(G.workspace_bytes, dtype=torch.uint8, device="cuda")
    res = {}
    for mode in ("1", "0"):
        G.set_option("graphs", int(mode))
        f = torch.full(G.f_shape, 1.0, device="cuda")
        G.osem(f, y, r, b1s, allpix, offs, 1e-3, None, 2, ws)
        G.osem(f, y, r, b1s, allpix, offs, 1e-3, None, 1, ws)   # replay of the cached graph
        G.osem(f, y, r, b1s, allpix, offs, 2e-3, None, 1, ws)   # new beta: re-capture
        torch.cuda.synchronize()
        res[mode] = f.clone()
    assert torch.equal(res["1"], res["0"])
    G.close()


@pytest.mark.parametrize("ci", [1, 2])
def test_launch_count_matches_kernels(ci):
    """cacsi_last_launch_count (bench.py's gpu_launches) equals the number of
    libcacsi kernel launches the per-kernel event timer saw, for the operators
    and the fused iteration (device and host-buffer entry points)."""
    cfg = make_config(ci)
    G = P.Geometry(cfg.desc())
    rng = np.random.default_rng(2)
    f = torch.as_tensor(cfg.f).cuda()
    g = torch.empty(G.g_shape, device="cuda")
    b = torch.empty(G.f_shape, device="cuda")
    y = torch.as_tensor(rng.poisson(20.0, G.g_shape).astype(np.float32)).cuda()
    r = torch.full(G.g_shape, 1.0, device="cuda")
    b1 = torch.as_tensor(rng.uniform(1.0, 2.0, G.f_shape).astype(np.float32)).cuda()
    ws = torch.empty(G.workspace_bytes, dtype=torch.uint8, device="cuda")
    host = [torch.as_tensor(t.cpu().numpy()).pin_memory() for t in (f, y, r, b1)]
    calls = {
        "forward": lambda: G.forward(f, g),
        "backward": lambda: G.backward(g, b),
        "iterate": lambda: G.iterate(f, y, r, b1, 1e-3, 1, ws),
        "iterate_host": lambda: G.iterate_host(host[0], host[1], host[2], host[3], 1e-3, 1),
    }
    G.forward(f, g)
    torch.cuda.synchronize()
    for name, call in calls.items():
        G.kernel_times()
        G.set_timing(True)
        call()
        torch.cuda.synchronize()
        G.set_timing(False)
        seen = sum(n for _, n in G.kernel_times().values())
        assert G.last_launch_count == seen, (name, G.last_launch_count, seen)
    G.close()
