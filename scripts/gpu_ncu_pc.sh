# ncu --set full with source of the two pair-cache kernels on config 2 (one launch each)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/npc_build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_pc_(fwd_v|bwd_tma)" -s 2 -c 2 \
  -o gpurun_out/npc_prof python scripts/quick_time.py --configs 2 --reps 2 > gpurun_out/npc_ncu.log 2>&1
echo rc=$?; tail -2 gpurun_out/npc_ncu.log
