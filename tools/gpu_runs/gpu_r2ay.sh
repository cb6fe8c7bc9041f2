# round 2: bench with the build's driver allocation time in the JSON (x2 to see the spread)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2; do
timeout 1200 python bench.py --no-cpu-baseline > gpurun_out/r2ay_bench_$i.json 2> gpurun_out/r2ay_bench_$i.err; echo bench_rc=$?
python -c "import json;d=json.load(open('gpurun_out/r2ay_bench_$i.json'));p=d['preprocessing'];print(d['value'], p['preprocessing_s'], p['component_apsp_s'], p['boundary_minus_k2_device_s'], p['driver_alloc'])"
done
