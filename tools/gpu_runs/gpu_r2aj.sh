# round 2: K2 row replication by NVLink peer reads (4 GPUs): sharded-build checks + bench K2 (IPC vs NCCL broadcasts)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29613"
timeout 600 $T tools/mgpu_check.py > gpurun_out/r2aj_mgpu.log 2>&1; echo mgpu_rc=$?
grep "bit-exact\|MISMATCH" gpurun_out/r2aj_mgpu.log
PSP_K2_FORCE_SPILL=1 timeout 600 $T tools/mgpu_check.py > gpurun_out/r2aj_mgpu_spill.log 2>&1; echo mgpu_spill_rc=$?
grep -c "bit-exact" gpurun_out/r2aj_mgpu_spill.log
timeout 1200 $T bench.py --gpus 4 --no-cpu-baseline > gpurun_out/r2aj_bench_n4.json 2> gpurun_out/r2aj_bench_n4.err; echo bench_rc=$?
python -c "import json;d=json.load(open('gpurun_out/r2aj_bench_n4.json'));p=d['preprocessing'];print('ipc', d['value'], p['preprocessing_s'], p['k2_device_s'], p['boundary_minus_k2_device_s'])"
PSP_K2_REPLICATE=nccl timeout 1200 $T bench.py --gpus 4 --no-cpu-baseline > gpurun_out/r2aj_bench_n4_nccl.json 2> gpurun_out/r2aj_bench_n4_nccl.err; echo bench_rc=$?
python -c "import json;d=json.load(open('gpurun_out/r2aj_bench_n4_nccl.json'));p=d['preprocessing'];print('nccl', d['value'], p['preprocessing_s'], p['k2_device_s'], p['boundary_minus_k2_device_s'])"
