# round 2: row-sharded storage on the f32 tolerance path (road grid), 2 GPUs
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29616"
timeout 1500 $T tools/row_storage_check.py --config road1m_k256 > gpurun_out/r2as_rows_road1m.log 2>&1; echo rc=$?
tail -2 gpurun_out/r2as_rows_road1m.log | cut -c1-700
