# round 2: the configs[1] line (Delaunay 262k, k=256) on 1 GPU with its CPU baseline
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python bench.py --config delaunay262k_k256 > gpurun_out/r2ar_bench_cfg2.json 2> gpurun_out/r2ar_bench_cfg2.err; echo bench_rc=$?
python -c "import json;d=json.load(open('gpurun_out/r2ar_bench_cfg2.json'));p=d['preprocessing'];r=d['roofline'];print(d['value'], d['e2e']['value'], r['frac'], r['executed_frac'], p['preprocessing_s'], p['k2_device_s'], d['cpu_baseline']['value'])"
