# round 2: closing full validation at HEAD (parallel CSR build/reorder, parallel recenter, kept winner)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/r2bw_pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/r2bw_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 python bench.py > gpurun_out/r2bw_bench.json 2> gpurun_out/r2bw_bench.err; echo bench_rc=$?
python -c "import json;d=json.load(open('gpurun_out/r2bw_bench.json'));p=d['preprocessing'];print(d['value'], d['e2e']['value'], d['roofline']['frac'], p['preprocessing_s'], p['boundary_minus_k2_device_s'], d['cpu_baseline']['value'])"
timeout 1500 python bench.py --impl reference > gpurun_out/r2bw_ref.json 2> gpurun_out/r2bw_ref.err; echo ref_rc=$?
python -c "import json;d=json.load(open('gpurun_out/r2bw_ref.json'));print(d['value'], d['preprocessing']['build_s'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2bw_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2bw_ncu_bench.log 2>&1; echo ncu_list_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:query_grouped --launch-skip 2 --launch-count 1 -o gpurun_out/r2bw_qg_cfg3 python tools/profile_query.py --config delaunay1m_k1024 --batches 4 > gpurun_out/r2bw_ncu.log 2>&1; echo ncu_rc=$?
