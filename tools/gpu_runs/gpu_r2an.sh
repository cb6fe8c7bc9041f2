# round 2: 4 GPUs after the rank-0 partition broadcast: bench, routed, row-storage, sharded-build checks
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29615"
timeout 1200 $T bench.py --gpus 4 --no-cpu-baseline > gpurun_out/r2an_bench_n4.json 2> gpurun_out/r2an_bench_n4.err; echo bench_rc=$?
python -c "import json;d=json.load(open('gpurun_out/r2an_bench_n4.json'));p=d['preprocessing'];print(d['value'], d['e2e']['value'], p['preprocessing_s'], p['partition_s'], p['k2_device_s'])"
timeout 900 $T tools/routed_check.py > gpurun_out/r2an_routed.log 2>&1; echo routed_rc=$?
grep -E "FAIL|routed_check|D:|D/packed" gpurun_out/r2an_routed.log | tail -10
timeout 600 $T tools/mgpu_check.py > gpurun_out/r2an_mgpu.log 2>&1; echo mgpu_rc=$?
grep "bit-exact\|MISMATCH" gpurun_out/r2an_mgpu.log
timeout 1200 $T tools/row_storage_check.py --config delaunay1m_k1024 > gpurun_out/r2an_rows_cfg3.log 2>&1; echo rows_rc=$?
tail -2 gpurun_out/r2an_rows_cfg3.log | cut -c1-900
