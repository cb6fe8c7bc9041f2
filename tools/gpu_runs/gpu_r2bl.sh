# round 2: 2- and 4-GPU benches after the FW-loop unroll (cfg3)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for N in 4 2; do
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2962$N bench.py --gpus $N --no-cpu-baseline > gpurun_out/r2bl_bench_n$N.json 2> gpurun_out/r2bl_bench_n$N.err; echo bench_rc=$?
python -c "import json;d=json.load(open('gpurun_out/r2bl_bench_n$N.json'));p=d['preprocessing'];print($N, d['value'], d['e2e']['value'], p['preprocessing_s'], p['partition_s'], p['k2_device_s'], p['k2_alu_frac_per_gpu'])"
done
