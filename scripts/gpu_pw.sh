# pcv_pw A/B on config 2 (bitwise tests first, then alternating bench runs)
TAG=${1:-pw}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
python -c "import paper_1603_06400_b200 as P; from workloads import make_config; G=P.Geometry(make_config(2).desc()); print(\"pc_segcap\", G.query(\"pc_segcap\"), \"esai_max_window\", G.query(\"esai_max_window\"))"; timeout 600 python -m pytest tests/test_gpu_determinism.py -q -k "pair_window or pipelined" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_pytest.log
bash scripts/sweep_opts.sh ${TAG} "pcv_pw=0" "pcv_pw=1" "pcv_pw=0" "pcv_pw=1"
