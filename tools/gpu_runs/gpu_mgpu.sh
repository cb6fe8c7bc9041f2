# 2/4-GPU driver for gpurun: sharded-build parity, routed queries, bench lines
N=${1:-2}
timeout 900 python -m pytest tests -m gpu -x -q -k "multigpu or routed or shard" > gpurun_out/pytest_mgpu.log 2>&1; echo pytest_exit=$? >> gpurun_out/pytest_mgpu.log
for cfg in delaunay262k_k256 delaunay1m_k1024; do
  PSP_FW_PROFILE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --config $cfg > gpurun_out/bench_${cfg}_n$N.json 2> gpurun_out/bench_${cfg}_n$N.err
done
