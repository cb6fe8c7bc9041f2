# round 2: 2 GPUs at HEAD (parallel CSR build/reorder, parallel recenter): bench N=2
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29615"
timeout 1200 $T bench.py --gpus 2 --no-cpu-baseline > gpurun_out/r2bz_bench_n2.json 2> gpurun_out/r2bz_bench_n2.err; echo bench_rc=$?
python -c "import json;d=json.load(open('gpurun_out/r2bz_bench_n2.json'));p=d['preprocessing'];print(d['value'], d['e2e']['value'], p['preprocessing_s'], p['partition_s'], p['k2_device_s'])"
