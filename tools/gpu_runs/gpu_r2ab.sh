# round 2: K2 working matrix reused as the block layout: parity + 4 repeated builds + bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/r2ab_parity.log 2>&1; echo parity_rc=$?
tail -1 gpurun_out/r2ab_parity.log
PSP_FW_PROFILE=1 timeout 900 python tools/build_repeat.py --config delaunay1m_k1024 --builds 4 > gpurun_out/r2ab_repeat.jsonl 2> gpurun_out/r2ab_repeat.err; echo rc=$?
grep "boundary lap: K2 done\|boundary lap: block\|K2 permutation" gpurun_out/r2ab_repeat.err | cut -c1-160
cat gpurun_out/r2ab_repeat.jsonl
timeout 1200 python bench.py --no-cpu-baseline > gpurun_out/r2ab_bench.json 2> gpurun_out/r2ab_bench.err; echo bench_rc=$?
python -c "import json;d=json.load(open('gpurun_out/r2ab_bench.json'));p=d['preprocessing'];print(d['value'], d['e2e']['value'], d['roofline']['frac'], p['preprocessing_s'], p['boundary_minus_k2_device_s'])"
