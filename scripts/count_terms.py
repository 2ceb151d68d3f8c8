"""Exact work counts per operator application (pairs, open pairs, effective
terms) for every config, from the ORACLE's counter only (oracle.count_terms).
Writes workloads/work_counts.json, which bench.py reads for its terms/s and
roofline arithmetic.   python scripts/count_terms.py"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from workloads import make_config  # noqa: E402

out = {}
for ci in range(5):
    cfg = make_config(ci)
    t0 = time.time()
    pairs, open_, terms = oracle.Geometry(cfg).count_terms()
    out[str(ci)] = {"name": cfg.name, "pairs": pairs, "open_pairs": open_, "effective_terms": terms,
                    "nominal_terms": pairs * cfg.ne, "open_fraction": open_ / pairs,
                    "effective_fraction": terms / (pairs * cfg.ne)}
    print(ci, out[str(ci)], f"{time.time() - t0:.1f}s", flush=True)
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "workloads", "work_counts.json")
json.dump(out, open(path, "w"), indent=1)
