# round 2: 16-bit residual query product: parity + bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "u16_residual or kernels_bitwise or large_boundaries or concurrent or sparse_grouping" 2>&1 | tail -15
timeout 1200 python bench.py --no-cpu-baseline > gpurun_out/r2r_bench.json 2> gpurun_out/r2r_bench.err; echo bench_rc=$?
python -c "import json;d=json.load(open('gpurun_out/r2r_bench.json'));p=d['preprocessing'];print(d['value'], d['e2e']['value'], d['roofline']['frac'], p['preprocessing_s'], p['boundary_minus_k2_device_s'])"
tail -3 gpurun_out/r2r_bench.err
