# round 2: ncu --set full of one mid-K2 fw_phase3 launch at cfg3 (source-level)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name regex:'fw_phase3' --launch-skip 1050 --launch-count 1 -o gpurun_out/r2be_p3 python tools/profile_query.py --config delaunay1m_k1024 --batches 1 > gpurun_out/r2be_ncu.log 2>&1; echo ncu_rc=$?
