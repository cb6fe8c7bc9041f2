# round 2: 1024-thread phase 1 for the boundary graph: parity + cfg3 K2 (wide vs narrow)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/r2ao_parity.log 2>&1; echo parity_rc=$?
tail -1 gpurun_out/r2ao_parity.log
timeout 900 python tools/build_repeat.py --config delaunay1m_k1024 --builds 2 > gpurun_out/r2ao_wide.jsonl 2>&1; echo rc=$?
grep k2_device gpurun_out/r2ao_wide.jsonl | cut -c1-200
PSP_FW_PHASE1_NARROW=1 timeout 900 python tools/build_repeat.py --config delaunay1m_k1024 --builds 2 > gpurun_out/r2ao_narrow.jsonl 2>&1; echo rc=$?
grep k2_device gpurun_out/r2ao_narrow.jsonl | cut -c1-200
