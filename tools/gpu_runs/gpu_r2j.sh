# round 2: 4-GPU K2 exchange A/B at cfg3 and cfg2, multi-GPU parity
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k multigpu 2>&1 | tail -2
for cfg in delaunay1m_k1024 delaunay262k_k256; do
for ex in p2p nccl; do
  PSP_K2_EXCHANGE=$ex PSP_FW_PROFILE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 4 --steps 5 --warmup 3 --no-cpu-baseline --config $cfg > gpurun_out/r2j_${cfg}_n4_$ex.json 2> gpurun_out/r2j_${cfg}_n4_$ex.err; echo $cfg $ex rc=$?
  grep -E "sharded FW nb=(1120|273)" gpurun_out/r2j_${cfg}_n4_$ex.err | head -4
  python -c "import json;d=json.load(open('gpurun_out/r2j_${cfg}_n4_$ex.json'));p=d['preprocessing'];print('$cfg $ex', d['value'], p['k2_device_s'], p['k2_alu_frac_per_gpu'], p['preprocessing_s'])"
done
done
