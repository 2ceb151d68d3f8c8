# the 8-byte (P-packed) default: DRAM traffic capture, GPU suite, bench
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/q8_build.log 2>&1
timeout 900 ncu --set full --clock-control none -k "regex:k_pc_(fwd_v|bwd_tma)|k_tc_gemm_(ar16|splitk16)" -c 4 \
  -o gpurun_out/q8_prof python scripts/quick_time.py --configs 2 --reps 1 > gpurun_out/q8_ncu.log 2>&1
python scripts/dram_traffic.py gpurun_out/q8_prof.ncu-rep gpurun_out/r2q8_dram_traffic.json > /dev/null 2>&1
cp gpurun_out/r2q8_dram_traffic.json profiles/r2q8_dram_traffic.json 2>/dev/null
timeout 1800 python -m pytest tests -m gpu -q -s > gpurun_out/q8_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/q8_pytest.log
tail -2 gpurun_out/q8_pytest.log
timeout 900 python bench.py > gpurun_out/q8_bench.json 2> gpurun_out/q8_bench.err
python - <<PY
import json
d=json.loads(open("gpurun_out/q8_bench.json").read().strip().splitlines()[-1])
print(d["ms_per_step"], {k:round(v["avg_ms"],4) for k,v in d["kernels"].items()}, d["roofline"], d["e2e"]["ms_per_step"], d["setup_ms"])
print(json.load(open("gpurun_out/r2q8_dram_traffic.json")))
PY
