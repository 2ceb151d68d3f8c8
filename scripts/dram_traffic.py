"""DRAM bytes per launch of the step's heavy kernels from an ncu --set full
capture, for bench.py's roofline "traffic" field.

    python scripts/dram_traffic.py gpurun_out/TAG_prof.ncu-rep profiles/r1s3_dram_traffic.json
"""
import csv
import io
import json
import subprocess
import sys

# ncu kernel name (prefix, template arguments stripped) -> bench.py's KScope name
NAMES = {"k_tc_gemm_ar": "k_tc_gemm_W", "k_tc_gemm_ar16": "k_tc_gemm_W", "k_pc_fwd_v": "k_pc_fwd", "k_pc_fwd": "k_pc_fwd",
         "k_pc_bwd_tma": "k_pc_bwd", "k_pc_bwd": "k_pc_bwd", "k_tc_gemm_splitk": "k_tc_gemm_b2",
         "k_tc_gemm_splitk16": "k_tc_gemm_b2"}
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    rep, out = sys.argv[1], sys.argv[2]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = {}
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].split("(")[0].split("<")[0].split("::")[-1].strip()
        if name.startswith("void "):
            name = name[5:]
        key = NAMES.get(name)
        if key is None or key in res:
            continue

        def val(m):
            return float(d[m].replace(",", "")) * UNIT.get(units[hdr.index(m)], 1.0)
        res[key] = {"ncu_kernel": name, "dram_read_bytes": val("dram__bytes_read.sum"),
                    "dram_write_bytes": val("dram__bytes_write.sum"), "ms": val("gpu__time_duration.sum") / 1e6
                    if units[hdr.index("gpu__time_duration.sum")] == "ns" else float(d["gpu__time_duration.sum"])}
    json.dump({"source": f"ncu --set full --clock-control none ({rep}); DRAM bytes per launch", "kernels": res},
              open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
