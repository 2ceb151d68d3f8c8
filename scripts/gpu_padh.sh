python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for o in pcb_padh=0 pc_perm_padh=1,pcb_padh=1 pc_perm_padh=1,pcb_padh=0 pcb_padh=0 pc_perm_padh=1,pcb_padh=1; do
  timeout 300 python scripts/quick_time.py --configs 2 --reps 20 --kernels --options $o > gpurun_out/ph2_t_$o.log 2>&1
  echo $o; head -1 gpurun_out/ph2_t_$o.log
done
for o in pc_perm_padh=1,pcb_padh=1 pcb_padh=0; do
timeout 600 ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,smsp__inst_executed_op_shared_atom.sum,gpu__time_duration.sum -k regex:"k_pc_(bwd_tma|fwd_v)" -s 4 -c 2 python scripts/quick_time.py --configs 2 --reps 1 --options $o 2>&1 | grep -E "k_pc|atom|op_ld|duration" | head -12
done
