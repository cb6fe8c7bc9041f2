# round 2: query product k-loop unrolled by 2 (A/B): parity + cfg3 timing
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_oracle_file.py -q -m gpu -x > gpurun_out/r2aw_parity.log 2>&1; echo parity_rc=$?
tail -1 gpurun_out/r2aw_parity.log
timeout 600 python tools/profile_query.py --config delaunay1m_k1024 --batches 12 > gpurun_out/r2aw_prof.log 2>&1; echo rc=$?
tail -1 gpurun_out/r2aw_prof.log | cut -c1-250
