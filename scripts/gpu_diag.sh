# A/B of a diagnostic build (conflict-free histogram atomics, wrong results) against the real one
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for i in 1 2; do
timeout 300 python scripts/quick_time.py --configs 2 --reps 20 --kernels > gpurun_out/diag_real_$i.log 2>&1; echo real; head -1 gpurun_out/diag_real_$i.log
cp paper_1603_06400_b200/libcacsi.so /tmp/real.so; cp scripts/diag/libcacsi_diag_atomics.so paper_1603_06400_b200/libcacsi.so
timeout 300 python scripts/quick_time.py --configs 2 --reps 20 --kernels > gpurun_out/diag_cf_$i.log 2>&1; echo conflict-free; head -1 gpurun_out/diag_cf_$i.log
cp /tmp/real.so paper_1603_06400_b200/libcacsi.so
done
