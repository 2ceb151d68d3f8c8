# targeted ncu sections (bank conflicts, issue, stalls, source counters) of the config-4 forward
# kernels: the default and each option string given
TAG=${1:-er4m}
shift
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
i=0
for o in "" "$@"; do
  timeout 900 ncu --section SchedulerStats --section WarpStateStats --section MemoryWorkloadAnalysis_Tables \
    --section ComputeWorkloadAnalysis --section LaunchStats --section Occupancy --section SourceCounters \
    --section InstructionStats --clock-control none --import-source on -k "regex:k_forward_(rec|lane|reg)" -c 1 \
    -o gpurun_out/${TAG}_$i python scripts/run_config4.py $o > gpurun_out/${TAG}_$i.log 2>&1
  echo "$i [$o] rc=$?"; i=$((i+1))
done
