"""Forward with the CTA-pair W GEMM vs the single-CTA one (dev check)."""
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
    f = torch.as_tensor(cfg.f).cuda()
    out = {}
    for mode in ("ar", "ar2"):
        G.set_option("wgemm", {"ar": 0, "ar2": 1}[mode])
        g = torch.empty(G.g_shape, device="cuda")
        G.forward(f, g)
        torch.cuda.synchronize()
        out[mode] = g.double().cpu().numpy()
    d = np.abs(out["ar"] - out["ar2"]).max() / np.abs(out["ar"]).max()
    print(ci, "max rel diff", d, "equal", np.array_equal(out["ar"], out["ar2"]), flush=True)
    G.close()
