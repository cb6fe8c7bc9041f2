# N-GPU: sharded-build parity (incl. forced spill), cfg4 / cfg3 / cfg2 bench lines with the FW profile
N=${1:-4}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "multigpu or routed or shard" > gpurun_out/s4b_pytest_n$N.log 2>&1; echo pytest_exit=$? >> gpurun_out/s4b_pytest_n$N.log
for cfg in road4m_k512 delaunay1m_k1024 delaunay262k_k256; do
  PSP_FW_PROFILE=1 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --config $cfg > gpurun_out/s4b_${cfg}_n$N.json 2> gpurun_out/s4b_${cfg}_n$N.err
done
