# checked build (device bounds checks) over the energy-resolving tests, and compute-sanitizer
# memcheck / racecheck / synccheck over scripts/sanitize.py --quick
TAG=${1:-san}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
python -m paper_1603_06400_b200.build --checked > gpurun_out/${TAG}_buildc.log 2>&1
CACSI_CHECKED=1 timeout 1200 python -m pytest tests/test_gpu_er_direct.py tests/test_gpu_pair_cache.py -q -x > gpurun_out/${TAG}_checked_pytest.log 2>&1; echo rc=$? >> gpurun_out/${TAG}_checked_pytest.log
tail -2 gpurun_out/${TAG}_checked_pytest.log
# the checked library over the sanitize workloads too (compute-sanitizer itself is refused on the pool)
CACSI_CHECKED=1 timeout 900 python scripts/sanitize.py > gpurun_out/${TAG}_checked_sanitize.log 2>&1; echo "checked sanitize.py rc=$?"
for t in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $t --error-exitcode 9 python scripts/sanitize.py --quick > gpurun_out/${TAG}_${t}.log 2>&1; echo "$t rc=$?"; tail -2 gpurun_out/${TAG}_${t}.log
done
