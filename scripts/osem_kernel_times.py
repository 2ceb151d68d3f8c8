import os, sys, json
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1603_06400_b200 as P
from workloads import make_config
cfg = make_config(1)
G = P.Geometry(cfg.desc())
sub = P.binding.symmetric_subsets(cfg.det_nx, cfg.det_ny, 8, 16).ravel()
nsub = int(sub.max()) + 1
lists = [np.flatnonzero(sub == p).astype(np.int32) for p in range(nsub)]
offs = np.concatenate([[0], np.cumsum([len(x) for x in lists])]).astype(np.int32)
allpix = torch.as_tensor(np.concatenate(lists)).cuda()
ones = torch.ones(G.g_shape, device="cuda")
b1s = torch.empty((nsub,) + G.f_shape, device="cuda")
for p in range(nsub):
    G.backward_subset(ones, allpix[offs[p]:offs[p+1]], b1s[p])
f = torch.full(G.f_shape, 1.0, device="cuda")
y = torch.full(G.g_shape, 100.0, device="cuda"); r = torch.full(G.g_shape, 5.0, device="cuda")
ws = torch.empty(G.workspace_bytes, dtype=torch.uint8, device="cuda")
G.osem(f, y, r, b1s, allpix, offs, 1e-3, None, 1, ws)
torch.cuda.synchronize()
G.set_timing(True) if hasattr(G, "set_timing") else P.binding.lib().cacsi_set_timing(G.handle, 1)
G.osem(f, y, r, b1s, allpix, offs, 1e-3, None, 1, ws)
torch.cuda.synchronize()
print(json.dumps(G.kernel_times() if hasattr(G, "kernel_times") else "no kernel_times"))
