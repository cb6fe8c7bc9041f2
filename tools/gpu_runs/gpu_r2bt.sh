# round 2: 4 GPUs at HEAD after the parallel CSR build/reorder: bench N=4, GPU suite (multi-GPU tests enabled)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29615"
timeout 1200 $T bench.py --gpus 4 --no-cpu-baseline > gpurun_out/r2bt_bench_n4.json 2> gpurun_out/r2bt_bench_n4.err; echo bench_rc=$?
python -c "import json;d=json.load(open('gpurun_out/r2bt_bench_n4.json'));p=d['preprocessing'];print(d['value'], d['e2e']['value'], p['preprocessing_s'], p['partition_s'], p['k2_device_s'])"
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/r2bt_pytest_gpu_n4.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/r2bt_pytest_gpu_n4.log
