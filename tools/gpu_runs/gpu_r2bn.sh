# round 2: the configs[3] line (road-like 2048^2 grid, f32 tolerance path, k=512) on 1 GPU
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python bench.py --config road4m_k512 > gpurun_out/r2bn_bench_road4m.json 2> gpurun_out/r2bn_bench_road4m.err; echo bench_rc=$?
python -c "import json;d=json.load(open('gpurun_out/r2bn_bench_road4m.json'));p=d['preprocessing'];r=d['roofline'];print(d['value'], d['e2e']['value'], d['dtype'], r['frac'], r.get('executed_frac'), p['preprocessing_s'], p['partition_s'], p['k2_device_s'], (d.get('cpu_baseline') or {}).get('value'))"
