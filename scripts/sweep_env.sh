#!/bin/bash
# Time bench.py under several environment settings (kernel-variant sweeps).
# usage (on the GPU box): bash scripts/sweep_env.sh TAG "VAR=a VAR2=b" "VAR=c" ...
TAG=$1; shift
mkdir -p gpurun_out
for cfg in "$@"; do
  name=$(echo "$cfg" | tr ' =' '_-')
  env $cfg timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/${TAG}_${name}.json 2> gpurun_out/${TAG}_${name}.err
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
