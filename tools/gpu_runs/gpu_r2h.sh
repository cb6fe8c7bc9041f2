# round 2: P2P panel exchange for the row-sharded K2 at 2 GPUs
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi topo -m 2>&1 | head -5
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k multigpu 2>&1 | tail -3
for ex in p2p nccl; do
  PSP_K2_EXCHANGE=$ex PSP_FW_PROFILE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2h_cfg3_n2_$ex.json 2> gpurun_out/r2h_cfg3_n2_$ex.err; echo $ex rc=$?
  grep -E "sharded FW|K2 \(FW" gpurun_out/r2h_cfg3_n2_$ex.err | head -4
  python -c "import json;d=json.load(open('gpurun_out/r2h_cfg3_n2_$ex.json'));p=d['preprocessing'];print('$ex', d['value'], p['k2_device_s'], p['k2_alu_frac_per_gpu'], p['preprocessing_s'])"
done
