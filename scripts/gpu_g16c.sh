python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g16e_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_gemm16.py -q -x > gpurun_out/g16e_pytest.log 2>&1; echo rc=$? >> gpurun_out/g16e_pytest.log
tail -3 gpurun_out/g16e_pytest.log
for o in b2_rings=0 b2_rings=1 b2_rings=2 b2_rings=0 b2_rings=1 b2_rings=2; do
  timeout 300 python scripts/quick_time.py --configs 2 --reps 20 --kernels --options $o > gpurun_out/g16e_t_$o.log 2>&1
  echo $o; head -1 gpurun_out/g16e_t_$o.log
done
