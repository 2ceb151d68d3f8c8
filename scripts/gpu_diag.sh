# Upper bound of the backward's histogram-atomic conflicts: A/B of the real build against a
# diagnostic one whose atomics go to lane-spread, conflict-free bins (WRONG results; timing only).
set -e
python -m paper_1603_06400_b200.build > /dev/null
cp paper_1603_06400_b200/libcacsi.so /tmp/real.so
cp paper_1603_06400_b200/csrc/pair_cache.cuh /tmp/pair_cache.cuh.orig
sed -i 's|atomicAdd(hv + b, __float2int_rn(av) - x1);|atomicAdd(hist_s + (tid \& 31) + 64 * u, __float2int_rn(av) - x1);|; s|atomicAdd(hv + b + 1, x1);|atomicAdd(hist_s + (tid \& 31) + 64 * u + 32, x1);|' paper_1603_06400_b200/csrc/pair_cache.cuh
python -m paper_1603_06400_b200.build > /dev/null
cp paper_1603_06400_b200/libcacsi.so /tmp/diag.so
cp /tmp/pair_cache.cuh.orig paper_1603_06400_b200/csrc/pair_cache.cuh
set +e
for i in 1 2; do
  cp /tmp/real.so paper_1603_06400_b200/libcacsi.so
  timeout 300 python scripts/quick_time.py --configs 2 --reps 20 --kernels > gpurun_out/diag_real_$i.log 2>&1; echo real; head -1 gpurun_out/diag_real_$i.log
  cp /tmp/diag.so paper_1603_06400_b200/libcacsi.so
  timeout 300 python scripts/quick_time.py --configs 2 --reps 20 --kernels > gpurun_out/diag_cf_$i.log 2>&1; echo conflict-free; head -1 gpurun_out/diag_cf_$i.log
done
cp /tmp/real.so paper_1603_06400_b200/libcacsi.so
