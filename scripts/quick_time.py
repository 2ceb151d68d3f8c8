"""Quick CUDA-event timing of cacsi_forward / cacsi_backward per config (dev tool)."""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1603_06400_b200 as P  # noqa: E402
from workloads import make_config  # noqa: E402


def time_op(fn, reps):
    s = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record(s)
        fn()
        b.record(s)
    torch.cuda.synchronize()
    return sorted(a.elapsed_time(b) for a, b in ev)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--kernels", action="store_true", help="also print per-kernel averages (forward and backward)")
    ap.add_argument("--options", default=None, help="kernel-variant options (cacsi_geometry_create_ex)")
    args = ap.parse_args()
    out = {}
    for ci in [int(c) for c in args.configs.split(",")]:
        cfg = make_config(ci)
        import time
        t0 = time.perf_counter()
        G = P.Geometry(cfg.desc(), options=args.options)
        torch.cuda.synchronize()
        setup_ms = (time.perf_counter() - t0) * 1e3
        f = torch.as_tensor(cfg.f).cuda()
        g = torch.empty(G.g_shape, dtype=torch.float32, device="cuda")
        w = torch.rand(G.g_shape, dtype=torch.float32, device="cuda")
        b = torch.empty(G.f_shape, dtype=torch.float32, device="cuda")
        for _ in range(2):
            G.forward(f, g)
            G.backward(w, b)
        tf = time_op(lambda: G.forward(f, g), args.reps)
        tb = time_op(lambda: G.backward(w, b), args.reps)
        if args.kernels:
            G.kernel_times()
            G.set_timing(True)
            time_op(lambda: (G.forward(f, g), G.backward(w, b)), args.reps)
            G.set_timing(False)
            print(json.dumps({k: round(v[0] / max(v[1], 1), 4) for k, v in G.kernel_times().items()}), flush=True)
        pairs = cfg.n_vox * cfg.n_det
        out[ci] = dict(fwd_ms=tf[len(tf) // 2], bwd_ms=tb[len(tb) // 2], pairs=pairs, setup_ms=setup_ms,
                       options=args.options,
                       fwd_pairs_per_s=pairs / tf[len(tf) // 2] * 1e3, bwd_pairs_per_s=pairs / tb[len(tb) // 2] * 1e3,
                       **{k: G.query(k) for k in ("esai_breakpoints", "esai_max_window", "esai_lut_cells",
                                                  "esai_lut_slow_cells", "ts_rho", "pair_cache_records",
                                                  "er_cache_records")})
        print(json.dumps({ci: out[ci]}), flush=True)
        G.close()


if __name__ == "__main__":
    main()
