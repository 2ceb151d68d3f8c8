python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for o in pcb_pfl1=0 pcb_pfl1=1 pcb_pfl1=0 pcb_pfl1=1; do
  timeout 300 python scripts/quick_time.py --configs 2 --reps 20 --kernels --options $o > gpurun_out/pf_t_$o.log 2>&1
  echo $o; head -1 gpurun_out/pf_t_$o.log
done
for o in pcb_pfl1=0 pcb_pfl1=1; do
timeout 600 ncu --metrics l1tex__t_sector_hit_rate.pct,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,gpu__time_duration.sum -k regex:"k_pc_bwd_tma" -s 2 -c 1 python scripts/quick_time.py --configs 2 --reps 1 --options $o 2>&1 | grep -E "hit_rate|op_ld|duration" | head -4
done
