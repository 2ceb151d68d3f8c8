python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for o in pcb_ctas=0 pc_q8=1 pc_q8=1,pcb_carve=85 pc_q8=1,pcb_carve=80 pcb_ctas=0 pc_q8=1,pcb_carve=85; do
  timeout 300 python scripts/quick_time.py --configs 2 --reps 20 --kernels --options $o > gpurun_out/cv2_t_$o.log 2>&1
  echo $o; head -1 gpurun_out/cv2_t_$o.log
done
for o in pcb_ctas=0 pc_q8=1,pcb_carve=85; do
timeout 600 ncu --metrics l1tex__t_sector_hit_rate.pct,gpu__time_duration.sum,launch__shared_mem_config_size,sm__warps_active.avg.pct_of_peak_sustained_active -k regex:"k_pc_bwd_tma" -s 2 -c 1 python scripts/quick_time.py --configs 2 --reps 1 --options $o 2>&1 | grep -E "hit_rate|duration|config_size|warps_active" | head -4
done
