# geometry-create stage times on config 2 (five creations) and the kernel launch list of one creation
TAG=${1:-setup}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 600 python scripts/setup_time.py 2 5 > gpurun_out/${TAG}_stages.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
  python scripts/setup_time.py 2 1 > gpurun_out/${TAG}_ncu.log 2>&1
cat gpurun_out/${TAG}_stages.log
