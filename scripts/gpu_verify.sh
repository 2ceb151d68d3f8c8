# build, smoke, the whole GPU suite, the default bench line and the config-4 line (no reference arm)
TAG=${1:-verify}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 1200 python bench.py --config 4 --steps 3 --warmup 3 > gpurun_out/${TAG}_bench4.json 2> gpurun_out/${TAG}_bench4.err
tail -1 gpurun_out/${TAG}_smoke.log; tail -3 gpurun_out/${TAG}_pytest.log
python - <<PY
import json
for f in ["${TAG}_bench.json", "${TAG}_bench4.json"]:
    try:
        d = json.loads(open("gpurun_out/" + f).read().strip().splitlines()[-1])
        print(f, d.get("ms_per_step"), d.get("value"), (d.get("roofline") or {}).get("frac"), (d.get("e2e") or {}).get("ms_per_step"), d.get("forward_ms"), d.get("backward_ms"), d.get("setup_ms"))
    except Exception as e:
        print(f, "ERR", e)
PY
