python -c "import __graft_entry__ as g; g.build()" > gpurun_out/er_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_er_direct.py tests/test_gpu_parity.py -q -x -k "er or energy or config4 or full_size or adjoint" > gpurun_out/er_pytest.log 2>&1; echo rc=$? >> gpurun_out/er_pytest.log
tail -3 gpurun_out/er_pytest.log
for o in er_bwd_carry=1 er_bwd_carry=0; do
  timeout 600 python scripts/quick_time.py --configs 4 --reps 3 --kernels --options $o > gpurun_out/er_t_$o.log 2>&1
  echo $o; cat gpurun_out/er_t_$o.log | cut -c1-400
done
