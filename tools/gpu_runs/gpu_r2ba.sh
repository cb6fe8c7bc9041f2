# round 2: query-side buffers allocated before K2: alloc log + parity + bench x2
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
PSP_ALLOC_LOG=1 PSP_FW_PROFILE=1 timeout 1200 python bench.py --no-cpu-baseline --steps 3 > gpurun_out/r2ba_bench.json 2> gpurun_out/r2ba_bench.err; echo bench_rc=$?
grep "took\|component phase\|boundary lap\|K2 permutation" gpurun_out/r2ba_bench.err | cut -c1-200 | head -60
python -c "import json;d=json.load(open('gpurun_out/r2ba_bench.json'));p=d['preprocessing'];print(p['preprocessing_s'], p['component_apsp_s'], p['boundary_minus_k2_device_s'], p['driver_alloc'])"
