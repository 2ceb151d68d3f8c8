# ncu --set full of the default config-4 energy-resolving kernels (k_forward_lane, the cached
# k_backward_er_x); kernel replay, one launch of each
TAG=${1:-er4n}
KS=${2:-"k_forward_lane|k_backward_er_x"}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 600 python scripts/run_config4.py > gpurun_out/${TAG}_plain.log 2>&1; echo rc=$? >> gpurun_out/${TAG}_plain.log
timeout 1800 ncu --set full --clock-control none --import-source on -k "regex:${KS}" -c ${3:-2} \
  -o gpurun_out/${TAG}_prof python scripts/run_config4.py > gpurun_out/${TAG}_ncu.log 2>&1
echo rc=$?; tail -3 gpurun_out/${TAG}_ncu.log
