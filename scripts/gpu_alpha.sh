# k_forward_rec with alpha_k staged in shared memory: GPU suite, then config-4 timing
TAG=${1:-alpha}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_pytest.log
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench4.json 2> gpurun_out/${TAG}_bench4.err
python -c "
import json; d=json.loads(open('gpurun_out/${TAG}_bench4.json').read().strip().splitlines()[-1])
print('config4', d['ms_per_step'], 'fwd', d['forward_ms'], 'bwd', d['backward_ms'], {k: round(v['avg_ms'],3) for k,v in d['kernels'].items() if v['avg_ms']>1})"
