# config-2 work loop: build, pair-cache + determinism tests, quick timing with per-kernel averages
# (default and each option string), bench line
TAG=${1:-c2}
shift
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_pair_cache.py tests/test_gpu_determinism.py -q -x > gpurun_out/${TAG}_pytest.log 2>&1; echo rc=$? >> gpurun_out/${TAG}_pytest.log
tail -3 gpurun_out/${TAG}_pytest.log
for o in "" "$@"; do
  timeout 600 python scripts/quick_time.py --configs 2 --reps 20 --kernels ${o:+--options "$o"} > gpurun_out/${TAG}_qt_${o:-default}.log 2>&1; echo "[$o]"; tail -2 gpurun_out/${TAG}_qt_${o:-default}.log | cut -c1-260
done
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; python -c "
import json; d=json.loads(open('gpurun_out/${TAG}_bench.json').read().strip().splitlines()[-1]); print('bench', d['ms_per_step'], d['kernels'])"
