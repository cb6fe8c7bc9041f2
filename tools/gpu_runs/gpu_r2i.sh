# round 2: full GPU suite + smoke + bench (fence-free rb issue)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/r2i_pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/r2i_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1200 python bench.py --no-cpu-baseline > gpurun_out/r2i_bench.json 2> gpurun_out/r2i_bench.err; echo bench_rc=$?
python -c "import json;d=json.load(open('gpurun_out/r2i_bench.json'));print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['preprocessing']['preprocessing_s'], d['preprocessing']['k2_device_s'])"
