python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for rep in 1 2; do
for o in pc_q8=2 pc_win=256 pcb_carve=80 pcv_items=1 pcv_items=4 pcv_pf=2; do
  timeout 300 python scripts/quick_time.py --configs 2 --reps 20 --kernels --options $o > gpurun_out/sw_t_${o}_$rep.log 2>&1
  echo $o; head -1 gpurun_out/sw_t_${o}_$rep.log | cut -c1-150
done
done
