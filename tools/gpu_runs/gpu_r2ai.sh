# round 2: ncu --set full of the 16-bit product kernel (cfg3, pre-converted offsets)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
PSP_QUERY_U16=1 timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name regex:'query_grouped' --launch-skip 2 --launch-count 1 -o gpurun_out/r2ai_qg16 python tools/profile_query.py --config delaunay1m_k1024 --batches 4 > gpurun_out/r2ai_ncu.log 2>&1; echo ncu_rc=$?
