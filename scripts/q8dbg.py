import sys, os, torch, numpy as np, time
sys.path.insert(0, os.getcwd())
import paper_1603_06400_b200 as P
from workloads import make_config
for ci in (1, 2):
    cfg = make_config(ci)
    G8, G10 = P.Geometry(cfg.desc()), P.Geometry(cfg.desc(), options="pc_q8=0")
    print(ci, "bytes", G8.query("pair_cache_record_bytes"), G10.query("pair_cache_record_bytes"), flush=True)
    f = torch.as_tensor(cfg.f).cuda()
    w = torch.rand(G8.g_shape, device="cuda")
    out = {}
    for tag, G in (("q8", G8), ("q10", G10)):
        g = torch.empty(G.g_shape, device="cuda"); b = torch.empty(G.f_shape, device="cuda")
        for _ in range(2): G.forward(f, g); G.backward(w, b)
        torch.cuda.synchronize()
        G.set_timing(True)
        G.forward(f, g); G.backward(w, b)
        torch.cuda.synchronize()
        kt = G.kernel_times(); G.set_timing(False)
        out[tag] = (g.clone(), b.clone())
        print(tag, {k: round(v[0], 3) for k, v in kt.items()}, flush=True)
    dg = (out["q8"][0] - out["q10"][0]).abs().max() / out["q10"][0].abs().max()
    db = (out["q8"][1] - out["q10"][1]).abs().max() / out["q10"][1].abs().max()
    print(ci, "maxdiff fwd", float(dg), "bwd", float(db), flush=True)
