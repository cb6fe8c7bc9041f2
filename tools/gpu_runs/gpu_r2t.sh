cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "u16_residual or kernels_bitwise" 2>&1 | tail -3
PSP_QUERY_STATS=1 timeout 900 python tools/profile_query.py --config delaunay1m_k1024 --batches 3 2>&1 | tail -4
PSP_QUERY_U16=0 timeout 900 python tools/profile_query.py --config delaunay1m_k1024 --batches 3 2>&1 | tail -1
