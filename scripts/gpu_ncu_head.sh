# ncu evidence of the current code: launch lists of the bench commands (config 2 and config 4;
# gpu__time_duration.sum, --clock-control none) and --set full captures of the dominant kernels
# (config 2: k_pc_fwd_v, k_pc_bwd_tma; config 4: k_forward_rec, k_backward_er_x).
#   bash scripts/gpu_ncu_head.sh TAG   -> gpurun_out/TAG{2,4}_{launches.csv,prof.ncu-rep}
TAG=${1:-head}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
B="--steps 2 --warmup 3 --no-cpu-baseline --no-config3 --no-config4"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/${TAG}2_launches.csv python bench.py $B > gpurun_out/${TAG}2_launches.log 2>&1
echo "c2 launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_pc_(fwd_v|bwd_tma)" -s 2 -c 2 \
  -o gpurun_out/${TAG}2_prof python scripts/quick_time.py --configs 2 --reps 2 > gpurun_out/${TAG}2_prof.log 2>&1
echo "c2 full rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/${TAG}4_launches.csv python bench.py --config 4 $B > gpurun_out/${TAG}4_launches.log 2>&1
echo "c4 launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:k_(forward_rec|backward_er_x)" -c 2 \
  -o gpurun_out/${TAG}4_prof python scripts/run_config4.py > gpurun_out/${TAG}4_prof.log 2>&1
echo "c4 full rc=$?"
ls -la gpurun_out/ | grep ${TAG}
