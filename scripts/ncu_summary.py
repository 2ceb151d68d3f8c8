"""Summarise ncu outputs for profiles/: launch-list shares and key metrics of a
--set full capture.   python scripts/ncu_summary.py TAG [out.md]"""
import csv
import io
import os
import subprocess
import sys
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.sum", "sm__inst_executed_pipe_alu.sum", "sm__inst_executed_pipe_lsu.sum",
        "sm__inst_executed_pipe_xu.sum", "sm__inst_executed.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers", "sm__cycles_elapsed.avg",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = defaultdict(lambda: [0, 0.0])
    for d in data:
        k = d["Kernel Name"].replace("cacsi::<unnamed>::", "").split("(")[0]
        agg[k][0] += 1
        agg[k][1] += float(d["Metric Value"])
    tot = sum(v[1] for v in agg.values())
    lines = ["| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{k}` | {v[0]} | {v[1] / 1e6:.3f} | {100 * v[1] / tot:.2f}% |")
    return "\n".join(lines)


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u = rows[0], rows[1]
    out = []
    for v in rows[2:]:
        out.append(f"**{v[h.index('Kernel Name')].split('(')[0]}** grid {v[h.index('Grid Size')]} "
                   f"block {v[h.index('Block Size')]}\n")
        out.append("| metric | value | unit |\n|---|---|---|")
        for k in KEYS:
            if k in h:
                out.append(f"| {k} | {v[h.index(k)]} | {u[h.index(k)]} |")
        out.append("")
    return "\n".join(out)


if __name__ == "__main__":
    tag = sys.argv[1]
    d = "gpurun_out"
    parts = [f"# ncu summary {tag}\n"]
    if os.path.exists(f"{d}/{tag}_launches.csv"):
        parts += ["## Launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised)\n",
                  launches(f"{d}/{tag}_launches.csv"), ""]
    if os.path.exists(f"{d}/{tag}_prof.ncu-rep"):
        parts += ["## --set full capture\n", full(f"{d}/{tag}_prof.ncu-rep")]
    text = "\n".join(parts)
    if len(sys.argv) > 2:
        open(sys.argv[2], "w").write(text)
    print(text)
