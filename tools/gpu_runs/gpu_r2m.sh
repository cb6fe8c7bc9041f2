# round 2: K2 order planned during Phase 2; repeated builds; full-size parity incl. road4m (f32)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/build_repeat.py --config delaunay1m_k1024 --builds 3 2>&1 | tail -4 | tee gpurun_out/r2m_build_repeat.jsonl
timeout 1200 python -m pytest tests/test_large_configs.py -q -s -x 2>&1 | grep -E "config|passed|failed|Error" | tee gpurun_out/r2m_large.log
