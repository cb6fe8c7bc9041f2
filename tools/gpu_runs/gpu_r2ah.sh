# round 2: 16-bit product with pre-converted row offsets (group_bases16 writes them): parity + cfg3 timing
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "u16 or grouped or kernel" > gpurun_out/r2ah_parity.log 2>&1; echo parity_rc=$?
tail -2 gpurun_out/r2ah_parity.log
timeout 600 python tools/profile_query.py --config delaunay1m_k1024 --batches 12 > gpurun_out/r2ah_u32.log 2>&1; echo rc=$?
tail -1 gpurun_out/r2ah_u32.log | cut -c1-300
PSP_QUERY_U16=1 PSP_QUERY_STATS=1 timeout 600 python tools/profile_query.py --config delaunay1m_k1024 --batches 12 > gpurun_out/r2ah_u16.log 2>&1; echo rc=$?
grep "16-bit product" gpurun_out/r2ah_u16.log | tail -2
tail -1 gpurun_out/r2ah_u16.log | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name regex:'group|query' --csv --log-file gpurun_out/r2ah_u16_launches.csv env PSP_QUERY_U16=1 python tools/profile_query.py --config delaunay1m_k1024 --batches 3 > /dev/null 2>&1; echo ncu_rc=$?
python tools/launch_summary.py gpurun_out/r2ah_u16_launches.csv | head -12
