# as gpu_variants.sh, plus the energy-resolving GPU tests under each variant
TAG=${1:-vt}
shift
L=paper_1603_06400_b200/libcacsi.so
cp $L /tmp/libcacsi_default.so
for v in "$@"; do
  cp paper_1603_06400_b200/libcacsi_$v.so $L
  timeout 600 python -m pytest tests/test_gpu_er_direct.py -q -x 2>&1 | tail -1
  timeout 600 python scripts/quick_time.py --configs 4 --reps 3 --kernels > gpurun_out/${TAG}_$v.log 2>&1; echo $v; head -1 gpurun_out/${TAG}_$v.log | cut -c1-120
done
cp /tmp/libcacsi_default.so $L
