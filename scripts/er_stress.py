"""Repeatability stress of the energy-resolving operators at full size (config 4): N forward +
backward repetitions compared bit for bit with the first (the record-fed forward's barrier-free
chunk protocol and the backward's prefetching).   python scripts/er_stress.py [N]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1603_06400_b200 as P  # noqa: E402
from workloads import make_config  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
cfg = make_config(4)
G = P.Geometry(cfg.desc())
assert G.query("er_fcache_records") > 0 and G.query("er_vcache_records") > 0
f = torch.as_tensor(cfg.f).cuda()
w = torch.as_tensor(np.random.default_rng(7).uniform(0, 1, G.g_shape).astype(np.float32)).cuda()
g0, b0 = torch.empty(G.g_shape, device="cuda"), torch.empty(G.f_shape, device="cuda")
G.forward(f, g0)
G.backward(w, b0)
bad = 0
for i in range(n):
    g, b = torch.empty_like(g0), torch.empty_like(b0)
    G.forward(f, g)
    G.backward(w, b)
    ok = torch.equal(g, g0) and torch.equal(b, b0)
    bad += not ok
    print(i, "ok" if ok else "DIFF", flush=True)
print(f"config 4: {n} repetitions, {bad} differing")
sys.exit(1 if bad else 0)
