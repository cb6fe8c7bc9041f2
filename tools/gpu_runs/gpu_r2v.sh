# round 2: row-sharded boundary-graph storage on 2 GPUs (routed parity incl. storage mode D,
# the replicated multi-GPU build regression, full-size cfg2 + cfg3 row storage vs Dijkstra)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T="python -m torch.distributed.run --standalone --nproc-per-node 2"
timeout 900 $T tools/routed_check.py > gpurun_out/r2v_routed.log 2>&1; echo routed_rc=$?
grep -E "FAIL|ok|D" gpurun_out/r2v_routed.log | tail -12
timeout 600 $T tools/mgpu_check.py > gpurun_out/r2v_mgpu.log 2>&1; echo mgpu_rc=$?
tail -3 gpurun_out/r2v_mgpu.log
timeout 900 $T tools/row_storage_check.py --config delaunay262k_k256 > gpurun_out/r2v_rows_cfg2.log 2>&1; echo rows_cfg2_rc=$?
tail -4 gpurun_out/r2v_rows_cfg2.log
timeout 1200 $T tools/row_storage_check.py --config delaunay1m_k1024 > gpurun_out/r2v_rows_cfg3.log 2>&1; echo rows_cfg3_rc=$?
tail -4 gpurun_out/r2v_rows_cfg3.log
