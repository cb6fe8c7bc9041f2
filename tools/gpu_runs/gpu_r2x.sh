# round 2: query_cta at 1K pairs on cfg3: timing + ncu --set full of one launch
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/profile_query.py --config delaunay1m_k1024 --batch 1000 --batches 50 --kernel cta > gpurun_out/r2x_cta1k.log 2>&1; echo rc=$?
tail -3 gpurun_out/r2x_cta1k.log
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:query_cta --launch-skip 5 --launch-count 1 -o gpurun_out/r2x_cta1k python tools/profile_query.py --config delaunay1m_k1024 --batch 1000 --batches 8 --kernel cta > gpurun_out/r2x_ncu.log 2>&1; echo ncu_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2x_launches_1k.csv python tools/profile_query.py --config delaunay1m_k1024 --batch 1000 --batches 8 --kernel cta > gpurun_out/r2x_ncu2.log 2>&1; echo ncu2_rc=$?
