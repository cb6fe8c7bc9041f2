# round 2: stream-ordered pool for large blocks; query product row split; full suite
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/build_repeat.py --config delaunay1m_k1024 --builds 3 2>&1 | tail -4 | tee gpurun_out/r2n_build_repeat.jsonl
timeout 1200 python bench.py --no-cpu-baseline > gpurun_out/r2n_bench.json 2> gpurun_out/r2n_bench.err; echo bench_rc=$?
python -c "import json;d=json.load(open('gpurun_out/r2n_bench.json'));p=d['preprocessing'];print(d['value'], d['e2e']['value'], d['roofline']['frac'], p['preprocessing_s'], p['k2_device_s'], p['boundary_minus_k2_device_s'])"
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/r2n_pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/r2n_pytest_gpu.log
