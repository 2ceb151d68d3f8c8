"""Brief of an ncu report (time, instructions, issue, shared wavefronts / conflicts, top stalls):
python scripts/ncu_brief.py report.ncu-rep [...]"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__sass_inst_executed_op_shared_ld.sum", "smsp__sass_inst_executed_op_global_ld.sum",
        "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "dram__bytes_read.sum"]
for path in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    for d in rows[2:]:
        print("====", path, d[hdr.index("Kernel Name")][:60])
        for k in KEYS:
            if k in hdr:
                print("  ", k, d[hdr.index(k)])
        st = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio")]
        sv = sorted(((float(d[hdr.index(h)] or 0), h) for h in st), reverse=True)[:7]
        print("   stalls/issue", [(h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""),
                                    round(v, 2)) for v, h in sv])
