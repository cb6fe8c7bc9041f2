# round 2: bench with the executed-relaxation model in the roofline entry
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python bench.py --no-cpu-baseline > gpurun_out/r2am_bench.json 2> gpurun_out/r2am_bench.err; echo bench_rc=$?
python -c "import json;d=json.load(open('gpurun_out/r2am_bench.json'));r=d['roofline'];print(d['value'], r['frac'], r['executed_frac'], r['useful_share_of_executed'])"
