# K1 component sharding check (2 GPUs) + 1-GPU K2 timing variance
timeout 900 python -m pytest tests -m gpu -x -q -k "multigpu or routed or shard" > gpurun_out/s3b_pytest_mgpu.log 2>&1; echo pytest_exit=$? >> gpurun_out/s3b_pytest_mgpu.log
for i in 1 2; do
PSP_FW_PROFILE=1 timeout 400 python bench.py --no-cpu-baseline > gpurun_out/s3b_cfg2_n1_$i.json 2> gpurun_out/s3b_cfg2_n1_$i.err
done
PSP_FW_PROFILE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 > gpurun_out/s3b_cfg2_n2.json 2> gpurun_out/s3b_cfg2_n2.err
PSP_FW_PROFILE=1 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --config road4m_k512 > gpurun_out/s3b_cfg4_n2.json 2> gpurun_out/s3b_cfg4_n2.err
