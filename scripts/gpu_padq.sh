python -c "import __graft_entry__ as g; g.build()" > gpurun_out/pq_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_pair_cache.py tests/test_gpu_determinism.py tests/test_gpu_parity.py -q -x > gpurun_out/pq_pytest.log 2>&1; echo rc=$? >> gpurun_out/pq_pytest.log
tail -3 gpurun_out/pq_pytest.log
for o in pcv_padq=1 pcv_padq=0 pcv_padq=1 pcv_padq=0; do
  timeout 300 python scripts/quick_time.py --configs 2 --reps 20 --kernels --options $o > gpurun_out/pq_t_$o.log 2>&1
  echo $o; head -1 gpurun_out/pq_t_$o.log
done
