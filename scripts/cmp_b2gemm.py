"""Backward with the B-multicast split-K GEMM vs without (dev check)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1603_06400_b200 as P  # noqa: E402
from workloads import make_config  # noqa: E402

for ci in (0, 1, 2):
    cfg = make_config(ci)
    G = P.Geometry(cfg.desc())
    w = torch.as_tensor(np.random.default_rng(1).uniform(0, 1, G.g_shape).astype(np.float32)).cuda()
    out = {}
    for mode in ("0", "1"):
        os.environ["CACSI_B2_MC"] = mode
        b = torch.empty(G.f_shape, device="cuda")
        G.backward(w, b)
        torch.cuda.synchronize()
        out[mode] = b.double().cpu().numpy()
    print(ci, "equal", np.array_equal(out["0"], out["1"]), float(np.abs(out["0"] - out["1"]).max()), flush=True)
    G.close()
