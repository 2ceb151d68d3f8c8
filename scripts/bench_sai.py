"""Scatter-angle interpolation (Table I row SAI) on config 2:
time of the SAI forward / backward against the exact operators and their
NRMSE (RMSE over the RMS of the exact result): forward on the
phantom, backward on the noiseless data g = A f, as in Table I.

    python scripts/bench_sai.py [--config 2] [--n 125,250,500,1000,2000] > out.json
"""
import argparse
import json
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1603_06400_b200 as P  # noqa: E402
from workloads import make_config  # noqa: E402


def timed(fn, reps=5):
    s = torch.cuda.current_stream()
    fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--n", default="125,250,500,1000,2000")
    args = ap.parse_args()
    cfg = make_config(args.config)
    f = torch.as_tensor(cfg.f).cuda()
    out = {"workload": cfg.name, "theta_range_rad": [0.2 * math.pi / 180, math.pi / 6], "rows": []}
    E = P.Geometry(cfg.desc())
    g = torch.empty(E.g_shape, dtype=torch.float32, device="cuda")
    b = torch.empty(E.f_shape, dtype=torch.float32, device="cuda")
    E.forward(f, g)
    data = g.clone()
    E.backward(data, b)
    g_ex, b_ex = g.double().cpu().numpy(), b.double().cpu().numpy()
    out["exact"] = {"fwd_ms": timed(lambda: E.forward(f, g)), "bwd_ms": timed(lambda: E.backward(data, b)),
                    "breakpoints": E.query("esai_breakpoints")}
    E.close()
    for n in [int(x) for x in args.n.split(",")]:
        d = cfg.desc()
        d.update(sai_n_theta=n, sai_theta_min=0.2 * math.pi / 180, sai_theta_max=math.pi / 6)
        G = P.Geometry(d)
        G.forward(f, g)
        G.backward(data, b)
        torch.cuda.synchronize()
        ef = float(np.linalg.norm(g.double().cpu().numpy() - g_ex) / np.linalg.norm(g_ex))
        eb = float(np.linalg.norm(b.double().cpu().numpy() - b_ex) / np.linalg.norm(b_ex))
        out["rows"].append({"n_theta": n, "cells": G.query("esai_breakpoints") - 1,
                            "fwd_ms": timed(lambda: G.forward(f, g)), "bwd_ms": timed(lambda: G.backward(data, b)),
                            "nrmse_fwd": ef, "nrmse_bwd": eb})
        G.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
