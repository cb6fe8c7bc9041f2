# round 2: f32 K2 with the unrolled tile loop (road4m full-size parity + K2 time)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/large_configs.jsonl
PSP_LARGE_CONFIGS=road4m_k512,delaunay262k_k256 timeout 1500 python -m pytest tests/test_large_configs.py -q -m gpu -x > gpurun_out/r2bg.log 2>&1; echo rc=$?
tail -1 gpurun_out/r2bg.log
grep -o '"config": "[a-z0-9_]*"\|"k2_device_s": [0-9.]*\|"mismatches": [0-9]*\|"max_rel_err": [0-9.e-]*' gpurun_out/large_configs.jsonl
