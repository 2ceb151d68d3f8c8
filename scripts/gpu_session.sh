#!/bin/bash
# One gpurun session: tests, bench, ncu launch list + one full capture.
# usage (on the GPU box): bash scripts/gpu_session.sh TAG [stages]
TAG=${1:-r}
STAGES=${2:-"test bench ncu"}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $OUT/${TAG}_smi.txt
echo "nproc=$(nproc)" >> $OUT/${TAG}_smi.txt
if [[ $STAGES == *test* ]]; then
  timeout 2400 python -m pytest tests -m gpu -q -s > $OUT/${TAG}_pytest.log 2>&1; echo "rc=$?" >> $OUT/${TAG}_pytest.log
fi
if [[ $STAGES == *bench* ]]; then
  timeout 600 python bench.py > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err; echo "rc=$?" >> $OUT/${TAG}_bench.err
fi
if [[ $STAGES == *micro* ]]; then
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/smem_atomic scripts/micro/smem_atomic.cu && /tmp/smem_atomic > $OUT/${TAG}_micro.log 2>&1
fi
if [[ $STAGES == *ncu* ]]; then
  CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
  timeout 600 $CMD > $OUT/${TAG}_ncu_plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_launches.csv $CMD > $OUT/${TAG}_ncu_launch.log 2>&1
  echo "launch rc=$?" >> $OUT/${TAG}_ncu_launch.log
  KREGEX=${KREGEX:-k_backward}
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$KREGEX" -s ${NCU_SKIP:-2} -c ${NCU_COUNT:-1} -o $OUT/${TAG}_prof $CMD > $OUT/${TAG}_ncu_full.log 2>&1
  echo "full rc=$?" >> $OUT/${TAG}_ncu_full.log
fi
