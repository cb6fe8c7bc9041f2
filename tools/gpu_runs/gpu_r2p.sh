# round 2: query_cta on the block layout by column quads x row phases
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "kernels_bitwise or point_query or sparse_grouping or large_boundaries" 2>&1 | tail -2
for args in "44 44 200000" "256 256 50000"; do PSP_SERVER_PROFILE=1 timeout 300 ./tools/latency_probe $args 2>&1; done | tee gpurun_out/r2p_latency.log
timeout 1500 python tools/query_sweep.py --config delaunay1m_k1024 --sizes 1e3,3e3,1e4,3e4,1e5,3e5 --kernels cta,grouped --no-e2e > gpurun_out/r2p_sweep.jsonl 2> gpurun_out/r2p_sweep.err; cat gpurun_out/r2p_sweep.jsonl | cut -c1-200
timeout 900 ./oracle/_ref/shim/gpu_acceptance > gpurun_out/r2p_acceptance.log 2>&1; echo acc_rc=$?; grep -E "criterion (1|9):|criteria" gpurun_out/r2p_acceptance.log
