cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
PSP_QUERY_STATS=1 timeout 900 python tools/profile_query.py --config delaunay1m_k1024 --batches 3 2>&1 | tail -5
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --kernel-name regex:"query_grouped|query_fallback|group_finish" --log-file gpurun_out/r2s_list.csv python tools/profile_query.py --config delaunay1m_k1024 --batches 3 > /dev/null 2>&1; echo ncu=$?
grep -E "query_grouped|query_fallback|group_finish" gpurun_out/r2s_list.csv | cut -c1-200 | tail -8
