# ncu --set full of the config-4 energy-resolving kernels (one forward, one backward; the
# create-time backward of ones is skipped); application replay (the kernels allocate per call)
TAG=${1:-erxn}
KS=${2:-"k_forward_reg|k_backward_er_x"}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 1500 ncu --set full --replay-mode application --clock-control none --import-source on -k "regex:${KS}" -s ${3:-1} -c ${4:-2} \
  -o gpurun_out/${TAG}_prof python scripts/run_config4.py > gpurun_out/${TAG}_ncu.log 2>&1
echo rc=$?; tail -2 gpurun_out/${TAG}_ncu.log
