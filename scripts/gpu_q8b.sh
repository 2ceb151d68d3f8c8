python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for rep in 1 2 3; do
for o in pc_q8=0 pc_q8=2 pc_q8=1; do
  timeout 300 python scripts/quick_time.py --configs 2 --reps 20 --kernels --options $o > gpurun_out/q8c_t_${o}_$rep.log 2>&1
  echo $o; head -1 gpurun_out/q8c_t_${o}_$rep.log
done
done
