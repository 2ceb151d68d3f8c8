# config-4 work loop: build, the energy-resolving GPU tests, quick timing (default and A/B options)
TAG=${1:-er4}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_er_direct.py -q -x > gpurun_out/${TAG}_pytest.log 2>&1; echo rc=$? >> gpurun_out/${TAG}_pytest.log
tail -3 gpurun_out/${TAG}_pytest.log
timeout 600 python scripts/quick_time.py --configs 4 --reps 3 --kernels > gpurun_out/${TAG}_qt.log 2>&1; tail -4 gpurun_out/${TAG}_qt.log
shift
for o in "$@"; do
  timeout 600 python scripts/quick_time.py --configs 4 --reps 3 --kernels --options "$o" > gpurun_out/${TAG}_qt_$o.log 2>&1; echo "$o"; tail -4 gpurun_out/${TAG}_qt_$o.log
done
