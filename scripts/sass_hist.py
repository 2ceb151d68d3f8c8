"""Opcode histogram of an ncu --page source --print-source sass CSV export.
    python scripts/sass_hist.py src.csv [top]"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = None
data = []
for r in rows:
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0].startswith("0x"):
        data.append(dict(zip(hdr, r)))
num = lambda x: int(x) if x and x.isdigit() else 0  # noqa: E731
tot = sum(num(d["Instructions Executed"]) for d in data)
samp = sum(num(d["Warp Stall Sampling (All Samples)"]) for d in data)
thr = sum(num(d["Thread Instructions Executed"]) for d in data)
print(f"warp inst {tot:.4e}  thread inst {thr:.4e}  samples {samp}")
c, s = Counter(), Counter()
for d in data:
    t = d["Source"].strip().split()
    if not t:
        continue
    op = t[1] if t[0].startswith("@") else t[0]
    op = ".".join(op.split(".")[:2]) if op.startswith(("ATOMS", "LDS", "LDG", "MUFU", "F2I", "I2F", "FRND")) else op.split(".")[0]
    c[op] += num(d["Instructions Executed"])
    s[op] += num(d["Warp Stall Sampling (All Samples)"])
for k, v in c.most_common(top):
    print(f"{k:14s} {v / tot * 100:6.2f}% inst  {s[k] / max(samp, 1) * 100:6.2f}% samples")
