# round 2: one-line mailbox; cta kernel on the block layout; u16 feasibility; ncu of query_grouped at cfg3
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for args in "44 44 200000" "44 1 200000" "256 256 50000"; do
  PSP_SERVER_PROFILE=1 timeout 300 ./tools/latency_probe $args 2>&1
done | tee gpurun_out/r2g_latency.log
timeout 600 python -m pytest tests -q -m gpu -x -k "point_query or kernels_bitwise or large_boundaries or concurrent" 2>&1 | tail -2
timeout 900 ./oracle/_ref/shim/gpu_acceptance > gpurun_out/r2g_acceptance.log 2>&1; echo acc_rc=$?
grep -E "criterion (1|9)|criteria" gpurun_out/r2g_acceptance.log
timeout 900 python tools/u16_feasibility.py --config delaunay1m_k1024 --components 16 2>&1 | tail -1 | tee gpurun_out/r2g_u16.json
timeout 1200 python tools/query_sweep.py --config delaunay1m_k1024 --sizes 1e3,1e4,3e4,1e5 --kernels cta,grouped --no-e2e > gpurun_out/r2g_sweep.jsonl 2> gpurun_out/r2g_sweep.err; cat gpurun_out/r2g_sweep.jsonl
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name regex:query_grouped --launch-skip 2 --launch-count 1 -o gpurun_out/r2g_qg_cfg3 python tools/profile_query.py --config delaunay1m_k1024 --batches 4 > gpurun_out/r2g_ncu.log 2>&1; echo ncu_rc=$?; tail -3 gpurun_out/r2g_ncu.log
