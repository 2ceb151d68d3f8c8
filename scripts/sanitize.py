"""Small workloads for compute-sanitizer (memcheck / initcheck / racecheck / synccheck):
every operator family on configs 0-1 through the C ABI, with a parity check so a run
that silently computes garbage also fails.

    compute-sanitizer --tool memcheck python scripts/sanitize.py [--quick]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1603_06400_b200 as P  # noqa: E402
from workloads import make_config  # noqa: E402


def run(G, f, w):
    g = torch.empty(G.g_shape, dtype=torch.float32, device="cuda")
    b = torch.empty(G.f_shape, dtype=torch.float32, device="cuda")
    G.forward(f, g)
    G.backward(w, b)
    torch.cuda.synchronize()
    return g, b


def main():
    quick = "--quick" in sys.argv
    cases = [(0, {}, None), (0, {}, "pair_cache=0"), (0, {}, "direct=1"), (0, dict(energy_resolving=1), None),
             (0, dict(energy_resolving=1), "er_cache=1"),
             (0, dict(sai_n_theta=250, sai_theta_min=0.0035, sai_theta_max=0.5236), None),
             # energy-resolving, several table chunks and voxel splits: the record-fed forward
             # (k_forward_rec, cp.async record ring, barrier-free chunk rounds) and the cached backward
             (0, dict(energy_resolving=1, ny=37, nz=41, det_nx=13, det_ny=29, ne=40,
                      energy_kev=np.linspace(21.0, 149.0, 40), phi=np.linspace(1.0, 0.3, 40), nq=33), None)]
    if not quick:
        cases += [(1, {}, None), (1, {}, "pair_cache=0")]
    rng = np.random.default_rng(0)
    for ci, over, opts in cases:
        cfg = make_config(ci)
        d = cfg.desc()
        d.update(over)
        G = P.Geometry(d, options=opts)
        f = torch.as_tensor(rng.random(G.f_shape, dtype=np.float32)).cuda()
        w = torch.as_tensor(rng.random(G.g_shape, dtype=np.float32)).cuda()
        g, b = run(G, f, w)
        # adjoint identity as a cheap correctness check
        lhs = float(torch.dot(g.double().ravel(), w.double().ravel()))
        rhs = float(torch.dot(f.double().ravel(), b.double().ravel()))
        assert abs(lhs - rhs) <= 1e-5 * abs(lhs), (ci, over, opts, lhs, rhs)
        if not d.get("energy_resolving"):
            ws = torch.empty(G.workspace_bytes, dtype=torch.uint8, device="cuda")
            y = torch.as_tensor(rng.poisson(20.0, G.g_shape).astype(np.float32)).cuda()
            r = torch.ones(G.g_shape, dtype=torch.float32, device="cuda")
            b1 = torch.empty(G.f_shape, dtype=torch.float32, device="cuda")
            G.backward(torch.ones_like(r), b1)
            fi = torch.ones(G.f_shape, dtype=torch.float32, device="cuda")
            G.iterate(fi, y, r, b1, 1e-3, 2, ws)
            fh = fi.cpu().numpy().copy()
            G.iterate_host(fh, y.cpu().numpy(), r.cpu().numpy(), b1.cpu().numpy(), 1e-3, 1)
            out = torch.zeros(1, dtype=torch.float64, device="cuda")
            G.neg_loglik(fi, y, r, 1e-3, out, ws)
            if ci == 0 and not over:
                sub = P.binding.symmetric_subsets(cfg.det_nx, cfg.det_ny, 2, 4).ravel()
                lists = [np.flatnonzero(sub == p).astype(np.int32) for p in range(int(sub.max()) + 1)]
                offs = np.concatenate([[0], np.cumsum([len(x) for x in lists])]).astype(np.int32)
                allpix = torch.as_tensor(np.concatenate(lists)).cuda()
                b1s = torch.empty((len(lists),) + G.f_shape, device="cuda")
                for p in range(len(lists)):
                    G.backward_subset(torch.ones_like(r), allpix[offs[p]:offs[p + 1]], b1s[p])
                G.osem(fi, y, r, b1s, allpix, offs, 1e-3, None, 1, ws)
            torch.cuda.synchronize()
        print("ok", ci, over, opts, flush=True)
        G.close()


if __name__ == "__main__":
    main()
