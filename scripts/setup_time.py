"""Geometry-create stage times (cacsi_query setup_us_*) for a config, N times in one process."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1603_06400_b200 as P  # noqa: E402
from workloads import make_config  # noqa: E402

KEYS = ("tables", "bitmaps", "bound", "pc_fill", "pc_perm", "pc_segwin", "host", "total")


def main():
    ci = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    opts = sys.argv[3] if len(sys.argv) > 3 else None
    cfg = make_config(ci)
    torch.cuda.init()
    for i in range(n):
        t0 = time.perf_counter()
        G = P.Geometry(cfg.desc(), options=opts)
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) * 1e3
        print(json.dumps({"run": i, "wall_ms": round(wall, 2), **{k: G.query("setup_us_" + k) / 1e3 for k in KEYS}}),
              flush=True)
        G.close()


if __name__ == "__main__":
    main()
