import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1603_06400_b200 as P
from workloads import make_config
for ci in (1, 3, 2):
    cfg = make_config(ci)
    G = P.Geometry(cfg.desc())
    rng = np.random.default_rng(5)
    for trial in range(3):
        w = torch.as_tensor(rng.uniform(0, 1, G.g_shape).astype(np.float32)).cuda()
        if trial == 2:
            w = torch.as_tensor(rng.uniform(0, 3000, G.g_shape).astype(np.float32)).cuda()
        outs = {}
        for mode in ("flat", "tma", "tma"):
            G.set_option("pc_bwd_flat", int(mode == "flat"))
            b = torch.empty(G.f_shape, device="cuda")
            G.backward(w, b)
            torch.cuda.synchronize()
            outs.setdefault(mode, []).append(b.cpu().numpy())
        f, t1, t2 = outs["flat"][0], outs["tma"][0], outs["tma"][1]
        print(ci, trial, "tma==flat", np.array_equal(f, t1), "tma==tma", np.array_equal(t1, t2),
              "maxdiff", float(np.abs(f - t1).max()), float(np.abs(f).max()))
    G.close()
