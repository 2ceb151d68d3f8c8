# time prebuilt library variants (paper_1603_06400_b200/libcacsi_<name>.so) on config 4 (and the default)
TAG=${1:-var}
shift
L=paper_1603_06400_b200/libcacsi.so
cp $L /tmp/libcacsi_default.so
timeout 600 python scripts/quick_time.py --configs ${CFG:-4} --reps 3 --kernels > gpurun_out/${TAG}_default.log 2>&1; echo default; head -1 gpurun_out/${TAG}_default.log | cut -c1-200
for v in "$@"; do
  cp paper_1603_06400_b200/libcacsi_$v.so $L
  timeout 600 python scripts/quick_time.py --configs ${CFG:-4} --reps 3 --kernels > gpurun_out/${TAG}_$v.log 2>&1; echo $v; head -1 gpurun_out/${TAG}_$v.log | cut -c1-200
done
cp /tmp/libcacsi_default.so $L
