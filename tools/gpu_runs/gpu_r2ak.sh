# round 2: clean 2-GPU bench (cfg3) + the configs[1] line on 2 GPUs
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29614"
timeout 1200 $T bench.py --gpus 2 --no-cpu-baseline > gpurun_out/r2ak_bench_n2.json 2> gpurun_out/r2ak_bench_n2.err; echo bench_rc=$?
python -c "import json;d=json.load(open('gpurun_out/r2ak_bench_n2.json'));p=d['preprocessing'];print(d['value'], d['e2e']['value'], p['preprocessing_s'], p['partition_s'], p['k2_device_s'], p['boundary_minus_k2_device_s'])"
timeout 1200 $T bench.py --gpus 2 --config delaunay262k_k256 --no-cpu-baseline > gpurun_out/r2ak_bench_cfg2_n2.json 2> gpurun_out/r2ak_bench_cfg2_n2.err; echo bench_rc=$?
python -c "import json;d=json.load(open('gpurun_out/r2ak_bench_cfg2_n2.json'));p=d['preprocessing'];print(d['value'], d['e2e']['value'], p['preprocessing_s'], p['k2_device_s'])"
