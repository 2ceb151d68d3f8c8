"""Reconstruction measurements on the config-3 problem (BASELINE.json configs[3]:
config-1 geometry, Poisson data with mean count 1e4 + background 5, beta = 1e-3,
uniform start): Alg. 5 EM (50 iterations, quadratic and Huber penalties) and
Alg. 6 OSEM with the paper's 64 symmetric subsets (rho_x = 8, rho_y = 16).
Reports time per (outer) iteration with CUDA events on the launching stream,
the objective J after each iteration (cacsi_neg_loglik_ex) and the final
relative error ||f - f_true|| / ||f_true||.  Every stage is a libcacsi call.

    python scripts/bench_recon.py [--iters 50] [--osem-outer 5] > out.json
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1603_06400_b200 as P  # noqa: E402
from workloads import make_config  # noqa: E402
from workloads.configs import seeded_rng  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--osem-outer", type=int, default=5)
    ap.add_argument("--huber-delta", type=float, default=0.02)
    args = ap.parse_args()
    cfg = make_config(1)
    G0 = P.Geometry(cfg.desc())
    f_true = torch.as_tensor(cfg.f).cuda()
    l_true = torch.empty(G0.g_shape, dtype=torch.float32, device="cuda")
    G0.forward(f_true, l_true)
    torch.cuda.synchronize()
    lt = l_true.double().cpu().numpy()
    s = 1e4 / lt.mean()
    G0.close()
    y_np = seeded_rng(3, 2).poisson(s * lt + 5.0).astype(np.float32)
    d = cfg.desc()
    d["scale"] = s
    G = P.Geometry(d)
    y = torch.as_tensor(y_np).cuda()
    r = torch.full(G.g_shape, 5.0, dtype=torch.float32, device="cuda")
    ones = torch.ones(G.g_shape, dtype=torch.float32, device="cuda")
    b1 = torch.empty(G.f_shape, dtype=torch.float32, device="cuda")
    G.backward(ones, b1)
    torch.cuda.synchronize()
    f0 = float((y_np - 5.0).sum() / b1.double().sum().item())
    ws = torch.empty(G.workspace_bytes, dtype=torch.uint8, device="cuda")
    jout = torch.zeros(1, dtype=torch.float64, device="cuda")
    beta = 1e-3
    stream = torch.cuda.current_stream()
    ft = f_true.double()

    def objective(f, pen):
        G.neg_loglik_ex(f, y, r, beta, pen, jout, ws)
        return jout.item()

    def relerr(f):
        return float(torch.linalg.norm(f.double() - ft) / torch.linalg.norm(ft))

    out = {"workload": "config3: config-1 geometry, Poisson mean 1e4 + r = 5, beta = 1e-3, uniform f0",
           "n_vox": cfg.n_vox, "n_det": cfg.n_det, "nq": cfg.nq, "ne": cfg.ne}
    for tag, pen in (("em_quadratic", None), ("em_huber", ("huber", args.huber_delta))):
        f = torch.full(G.f_shape, f0, dtype=torch.float32, device="cuda")
        G.iterate_ex(f, y, r, b1, beta, pen, 1, ws)  # warm-up (allocator, clocks)
        f.fill_(f0)
        trace = [objective(f, pen)]
        times = []
        for _ in range(args.iters):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            G.iterate_ex(f, y, r, b1, beta, pen, 1, ws)
            b.record(stream)
            torch.cuda.synchronize()
            times.append(a.elapsed_time(b))
            trace.append(objective(f, pen))
        out[tag] = {"ms_per_iter_median": float(np.median(times)), "iters": args.iters,
                    "objective": [trace[i] for i in (0, 1, 2, 5, 10, 20, len(trace) - 1) if i < len(trace)],
                    "objective_monotone": bool(all(b <= a * (1 + 1e-9) for a, b in zip(trace, trace[1:]))),
                    "final_rel_err_vs_f_true": relerr(f)}
        if tag == "em_quadratic":
            em_trace = trace
    # ---- OSEM, 64 symmetric subsets
    sub = P.binding.symmetric_subsets(cfg.det_nx, cfg.det_ny, 8, 16).ravel()
    nsub = int(sub.max()) + 1
    lists = [np.flatnonzero(sub == p).astype(np.int32) for p in range(nsub)]
    offs = np.concatenate([[0], np.cumsum([len(x) for x in lists])]).astype(np.int32)
    allpix = torch.as_tensor(np.concatenate(lists)).cuda()
    b1s = torch.empty((nsub,) + G.f_shape, dtype=torch.float32, device="cuda")
    for p in range(nsub):
        G.backward_subset(ones, allpix[offs[p]:offs[p + 1]], b1s[p])
    f = torch.full(G.f_shape, f0, dtype=torch.float32, device="cuda")
    G.osem(f, y, r, b1s, allpix, offs, beta, None, 1, ws)  # warm-up
    f.fill_(f0)
    trace = [objective(f, None)]
    times = []
    for _ in range(args.osem_outer):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        G.osem(f, y, r, b1s, allpix, offs, beta, None, 1, ws)
        b.record(stream)
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b))
        trace.append(objective(f, None))
    # EM iterations needed to reach each OSEM outer iterate's objective
    equiv = []
    for j in trace[1:]:
        k = next((i for i, v in enumerate(em_trace) if v <= j), None)
        equiv.append(k if k is not None else f">{len(em_trace) - 1}")
    out["osem_64"] = {"subsets": nsub, "ms_per_outer_iter_median": float(np.median(times)),
                      "objective": trace, "em_iters_to_match_each_outer_iter": equiv,
                      "final_rel_err_vs_f_true": relerr(f)}
    G.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
