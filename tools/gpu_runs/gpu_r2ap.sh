# round 2: phase-1 kernel durations (wide vs narrow) on the cfg3 boundary graph
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name regex:'fw_phase1' --launch-skip 200 --launch-count 30 --csv --log-file gpurun_out/r2ap_wide.csv python tools/profile_query.py --config delaunay1m_k1024 --batches 1 > /dev/null 2>&1; echo rc=$?
PSP_FW_PHASE1_NARROW=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name regex:'fw_phase1' --launch-skip 200 --launch-count 30 --csv --log-file gpurun_out/r2ap_narrow.csv python tools/profile_query.py --config delaunay1m_k1024 --batches 1 > /dev/null 2>&1; echo rc=$?
python tools/launch_summary.py gpurun_out/r2ap_wide.csv | head -4
python tools/launch_summary.py gpurun_out/r2ap_narrow.csv | head -4
