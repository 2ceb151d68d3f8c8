"""Top warp-stall-sampled SASS lines of an ncu report: python scripts/ncu_hot.py report [kernel-regex] [n]"""
import csv
import io
import subprocess
import sys

path = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else "."
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + kre],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ie, src = hdr.index("Instructions Executed"), hdr.index("Source")
smp = hdr.index("Warp Stall Sampling (All Samples)")
data = [r for r in rows[2:] if len(r) == len(hdr) and r[ie].isdigit()]
tot = sum(int(r[smp] or 0) for r in data)
print("samples", tot)
for i, r in sorted(enumerate(data), key=lambda x: -int(x[1][smp] or 0))[:n]:
    print(f"{i:5d} {int(r[smp]) / tot:6.3f} {int(r[ie]):>12d}  {r[src].strip()[:90]}")
