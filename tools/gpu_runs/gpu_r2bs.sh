# round 2: parallel host CSR build / reorder — GPU suite, smoke, bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/r2bs_pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/r2bs_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 python bench.py > gpurun_out/r2bs_bench.json 2> gpurun_out/r2bs_bench.err; echo bench_rc=$?
python -c "import json;d=json.load(open('gpurun_out/r2bs_bench.json'));p=d['preprocessing'];print(d['value'], d['e2e']['value'], d['roofline']['frac'], p)"
