#!/bin/bash
# Time bench.py under several kernel-variant option sets (cacsi_geometry_create_ex).
# usage (on the GPU box): bash scripts/sweep_opts.sh TAG "key=a,key2=b" "key=c" ...
TAG=$1; shift
mkdir -p gpurun_out
for cfg in "$@"; do
  name=$(echo "$cfg" | tr ',=' '_-')
  timeout 300 python bench.py --no-cpu-baseline --no-config3 --no-config4 --steps 20 --options "$cfg" > gpurun_out/${TAG}_${name}.json 2> gpurun_out/${TAG}_${name}.err
  python - "$cfg" gpurun_out/${TAG}_${name}.json >> gpurun_out/${TAG}_sweep.txt <<'PY'
import json, sys
try:
    d = json.load(open(sys.argv[2]))
    ks = {k: round(v["avg_ms"], 3) for k, v in d["kernels"].items() if v["avg_ms"] > 0.05}
    print(f"{sys.argv[1]:40s} step {d['ms_per_step']:.3f} fwd {d['forward_ms']:.3f} bwd {d['backward_ms']:.3f} {ks}")
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
done
cat gpurun_out/${TAG}_sweep.txt
