# ncu --set full of the two fp16-rate GEMMs on config 2 (one launch each)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/n16_build.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_tc_gemm_(ar16|splitk16)" -c 2 \
  -o gpurun_out/n16_gemm python scripts/quick_time.py --configs 2 --reps 1 > gpurun_out/n16_ncu.log 2>&1
echo rc=$?; tail -3 gpurun_out/n16_ncu.log
