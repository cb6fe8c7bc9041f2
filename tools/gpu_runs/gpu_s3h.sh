# 4-GPU lines: sharded-build parity, cfg2 / cfg3 / cfg4 bench (component-sharded ordered K1, packed K2)
N=${1:-4}
timeout 900 python -m pytest tests -m gpu -x -q -k "multigpu or routed or shard" > gpurun_out/s3h_pytest_mgpu_n$N.log 2>&1; echo pytest_exit=$? >> gpurun_out/s3h_pytest_mgpu_n$N.log
for cfg in delaunay262k_k256 delaunay1m_k1024 road4m_k512; do
  PSP_FW_PROFILE=1 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --config $cfg > gpurun_out/s3h_${cfg}_n$N.json 2> gpurun_out/s3h_${cfg}_n$N.err
done
