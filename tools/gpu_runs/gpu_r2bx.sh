# round 2: configs[3] (road4m, f32) at HEAD: full-size parity (Dijkstra) and the bench line with the parallel partitioner steps
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
PSP_LARGE_CONFIGS=road4m_k512 timeout 1500 python -m pytest tests/test_large_configs.py -q -m gpu -x > gpurun_out/r2bx_large.log 2>&1; echo large_rc=$?
tail -2 gpurun_out/r2bx_large.log
timeout 1500 python bench.py --config road4m_k512 > gpurun_out/r2bx_road4m.json 2> gpurun_out/r2bx_road4m.err; echo bench_rc=$?
python -c "import json;d=json.load(open('gpurun_out/r2bx_road4m.json'));p=d['preprocessing'];print(d['value'], d['e2e']['value'], d['roofline']['frac'], p['partition_s'], p['preprocessing_s'], p['k2_device_s'], d['cpu_baseline']['value'])"
