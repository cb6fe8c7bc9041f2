# round 2: sparse grouping parity + configs[4] batch sweep at cfg3 (1 GPU)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "sparse_grouping or kernels_bitwise or concurrent or point_query" 2>&1 | tail -2
timeout 1500 python tools/query_sweep.py --config delaunay1m_k1024 --sizes 1e3,1e4,1e5,1e6,1e7,1e8 --kernels auto > gpurun_out/r2k_sweep.jsonl 2> gpurun_out/r2k_sweep.err; echo sweep_rc=$?
cat gpurun_out/r2k_sweep.jsonl; tail -2 gpurun_out/r2k_sweep.err
