# fixed-point energy-resolving backward: tests + config-4 timing (both backward kernels)
TAG=${1:-erx}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_er_direct.py -q -x -s > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 900 python scripts/quick_time.py --configs 4 --reps 3 --kernels > gpurun_out/${TAG}_c4.log 2>&1
timeout 900 python scripts/quick_time.py --configs 4 --reps 3 --options er_bwd_fx=0 > gpurun_out/${TAG}_c4_old.log 2>&1
tail -3 gpurun_out/${TAG}_pytest.log; tail -2 gpurun_out/${TAG}_c4.log; tail -1 gpurun_out/${TAG}_c4_old.log
