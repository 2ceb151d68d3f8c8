# build, ER tests, config-4 quick timing, targeted ncu of the default forward
TAG=${1:-er4b}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_er_direct.py -q -x > gpurun_out/${TAG}_pytest.log 2>&1; echo rc=$? >> gpurun_out/${TAG}_pytest.log
tail -3 gpurun_out/${TAG}_pytest.log
timeout 600 python scripts/quick_time.py --configs 4 --reps 3 --kernels > gpurun_out/${TAG}_qt.log 2>&1; tail -4 gpurun_out/${TAG}_qt.log
timeout 900 ncu --section SchedulerStats --section WarpStateStats --section MemoryWorkloadAnalysis_Tables \
    --section ComputeWorkloadAnalysis --section LaunchStats --section Occupancy --section SourceCounters \
    --section InstructionStats --clock-control none --import-source on -k "regex:${2:-k_forward_rec}" -c 1 \
    -o gpurun_out/${TAG}_ncu python scripts/run_config4.py > gpurun_out/${TAG}_ncu.log 2>&1; echo ncu rc=$?
