# round 2: row-storage shard creation laps at 4 GPUs (cfg3)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29612"
PSP_FW_PROFILE=1 timeout 900 $T tools/row_storage_check.py --config delaunay1m_k1024 > gpurun_out/r2ad.log 2>&1; echo "rc=$?"
grep "shard lap" gpurun_out/r2ad.log
grep -o '"shard_create_s": \[[^]]*\]' gpurun_out/r2ad.log
