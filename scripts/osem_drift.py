"""Diagnostic: per-sub-iteration drift of GPU OSEM vs the fp64 oracle on the
config-3 problem (64 symmetric subsets).  Dev tool, not a test."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_1603_06400_b200 as P  # noqa: E402
from oracle import recon  # noqa: E402
from workloads import make_config  # noqa: E402
from workloads.configs import seeded_rng  # noqa: E402

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
sub = P.binding.symmetric_subsets(cfg.det_nx, cfg.det_ny, 8, 16).ravel()
lists = [np.flatnonzero(sub == p).astype(np.int32) for p in range(64)]
ones = torch.ones(G.g_shape, dtype=torch.float32, device="cuda")
b1_ref = O.backward(np.ones(O.g_shape))
f0 = np.full(G.f_shape, (y - r).sum() / b1_ref.sum(), dtype=np.float32)
f = torch.as_tensor(f0).cuda()
fr = f0.astype(np.float64)
yt, rt = torch.as_tensor(y).cuda(), torch.as_tensor(r).cuda()
l = torch.empty(G.g_shape, dtype=torch.float32, device="cuda")
b2 = torch.empty(G.f_shape, dtype=torch.float32, device="cuda")
b1p = torch.empty(G.f_shape, dtype=torch.float32, device="cuda")
fn = torch.empty_like(f)
beta = 1e-3 / 64
for p in range(64):
    pix = lists[p]
    pt = torch.as_tensor(pix).cuda()
    G.backward_subset(ones, pt, b1p)
    G.forward_subset(f, pt, l)
    G.ratio(l, yt, rt, l)
    G.backward_subset(l, pt, b2)
    G.update(f, b1p, b2, beta, fn)
    f.copy_(fn)
    torch.cuda.synchronize()
    # oracle step from ITS OWN previous iterate (drift) and from the GPU's iterate (one-step error)
    ind = np.zeros(O.g_shape).reshape(-1)
    ind[pix] = 1
    ind = ind.reshape(O.g_shape)
    b1r = O.backward_pixels(np.ones(O.g_shape), pix)
    gr = np.zeros(O.g_shape).reshape(-1)
    gr[pix] = O.forward_pixels(fr, pix)
    rat = recon.ratio(gr.reshape(O.g_shape), y, r) * ind
    fr = recon.update(fr, b1r, O.backward_pixels(rat, pix), beta)
    x = f.cpu().numpy().astype(np.float64)
    e = np.abs(x - fr) / np.maximum(np.abs(fr), 1e-30)
    sel = np.abs(fr) >= 1e-3 * np.abs(fr).max()
    k = np.unravel_index(np.argmax(np.where(sel, e, 0)), e.shape)
    if p % 8 == 0 or p == 63:
        print(f"sub {p:2d}: rel_l2 {np.linalg.norm(x - fr) / np.linalg.norm(fr):.3e} max_rel {e[sel].max():.3e} "
              f"at {k} f={fr[k]:.4e} b1p={b1r[k]:.3e} (max b1p {b1r.max():.3e})", flush=True)
