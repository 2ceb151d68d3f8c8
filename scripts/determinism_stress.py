"""Repeat the operators many times and check bitwise reproducibility (catches
races in the shared-memory staging / mbarrier rings).
    python scripts/determinism_stress.py [reps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1603_06400_b200 as P  # noqa: E402
from workloads import make_config  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
for ci in (1, 2):
    cfg = make_config(ci)
    G = P.Geometry(cfg.desc())
    f = torch.as_tensor(cfg.f).cuda()
    w = torch.as_tensor(np.random.default_rng(3).uniform(0, 1, G.g_shape).astype(np.float32)).cuda()
    g0 = torch.empty(G.g_shape, device="cuda")
    b0 = torch.empty(G.f_shape, device="cuda")
    G.forward(f, g0)
    G.backward(w, b0)
    torch.cuda.synchronize()
    bad_f = bad_b = 0
    for mode in ("flat", "tma"):
        G.set_option("pc_bwd_flat", int(mode == "flat"))
        for r in range(reps):
            g = torch.empty_like(g0)
            b = torch.empty_like(b0)
            G.forward(f, g)
            G.backward(w, b)
            torch.cuda.synchronize()
            if not torch.equal(g, g0):
                bad_f += 1
                d = (g - g0).abs()
                print(f"config {ci} rep {r}: forward differs at {int((d > 0).sum())} pixels, max {float(d.max()):.3e}")
            if not torch.equal(b, b0):
                bad_b += 1
                d = (b - b0).abs()
                print(f"config {ci} {mode} rep {r}: backward differs at {int((d > 0).sum())} entries, max {float(d.max()):.3e}")
    print(f"config {ci}: forward mismatches {bad_f}, backward mismatches {bad_b} over {2 * reps} reps")
    G.close()
