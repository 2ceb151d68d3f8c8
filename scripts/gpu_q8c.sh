python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_pair_cache.py tests/test_gpu_recon_ext.py tests/test_gpu_parity_full.py tests/test_gpu_gemm16.py -q -s 2>&1 | grep -E "8-byte|signed|log-uniform|all 65536|all 16384|passed|failed" | head -40
for rep in 1 2; do
for o in pc_q8=0 pc_q8=2; do
  timeout 300 python scripts/quick_time.py --configs 2 --reps 20 --kernels --options $o > gpurun_out/q8d_t_${o}_$rep.log 2>&1
  echo $o; head -1 gpurun_out/q8d_t_${o}_$rep.log
done
done
