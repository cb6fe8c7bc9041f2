# round 2: query-side buffers allocated before K2: parity, alloc log, bench x2
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_oracle_file.py -q -m gpu -x > gpurun_out/r2bb_parity.log 2>&1; echo parity_rc=$?
tail -1 gpurun_out/r2bb_parity.log
PSP_ALLOC_LOG=1 timeout 1200 python bench.py --no-cpu-baseline --steps 3 > gpurun_out/r2bb_bench0.json 2> gpurun_out/r2bb_bench0.err; echo bench_rc=$?
grep "took" gpurun_out/r2bb_bench0.err | head -20
for i in 1 2; do
timeout 1200 python bench.py --no-cpu-baseline > gpurun_out/r2bb_bench_$i.json 2> gpurun_out/r2bb_bench_$i.err; echo bench_rc=$?
python -c "import json;d=json.load(open('gpurun_out/r2bb_bench_$i.json'));p=d['preprocessing'];print(d['value'], p['preprocessing_s'], p['component_apsp_s'], p['boundary_minus_k2_device_s'], p['driver_alloc'])"
done
