python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g16b_build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/g16b_pytest.log 2>&1; echo rc=$? >> gpurun_out/g16b_pytest.log
tail -3 gpurun_out/g16b_pytest.log
for o in gemm16=0 b2_splits=8 b2_splits=12 b2_splits=16 b2_splits=24; do
  timeout 300 python scripts/quick_time.py --configs 2 --reps 20 --kernels --options $o > gpurun_out/g16b_t_$o.log 2>&1
  echo $o; head -1 gpurun_out/g16b_t_$o.log
done
timeout 600 python bench.py > gpurun_out/g16b_bench.json 2> gpurun_out/g16b_bench.err; tail -c 300 gpurun_out/g16b_bench.json
