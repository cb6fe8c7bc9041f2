# round 2: cross-task prefetch in query_grouped (QM_BLOCKS): parity + cfg3 bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/r2w_parity.log 2>&1; echo parity_rc=$?
tail -2 gpurun_out/r2w_parity.log
timeout 1200 python bench.py --no-cpu-baseline > gpurun_out/r2w_bench.json 2> gpurun_out/r2w_bench.err; echo bench_rc=$?
python -c "import json;d=json.load(open('gpurun_out/r2w_bench.json'));print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['ms_per_step'])"
