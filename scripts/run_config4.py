"""Run the config-4 (energy-resolving) forward and backward once each (ncu target).

    python scripts/run_config4.py [options]   (cacsi_geometry_create_ex kernel-variant options)"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1603_06400_b200 as P  # noqa: E402
from workloads import make_config  # noqa: E402

cfg = make_config(4)
G = P.Geometry(cfg.desc(), options=sys.argv[1] if len(sys.argv) > 1 else None)
f = torch.as_tensor(cfg.f).cuda()
g = torch.empty(G.g_shape, dtype=torch.float32, device="cuda")
b = torch.empty(G.f_shape, dtype=torch.float32, device="cuda")
G.forward(f, g)
w = torch.rand(G.g_shape, dtype=torch.float32, device="cuda")
G.backward(w, b)
torch.cuda.synchronize()
print("ok", float(g.double().sum()), float(b.double().sum()))
