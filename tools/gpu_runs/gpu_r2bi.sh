# round 2: FW min-plus tile loop unrolled by 8 k-pairs (A/B vs 4): parity + cfg3 K2 time
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/r2bi_parity.log 2>&1; echo parity_rc=$?
tail -1 gpurun_out/r2bi_parity.log
timeout 900 python tools/build_repeat.py --config delaunay1m_k1024 --builds 2 > gpurun_out/r2bi_repeat.jsonl 2>&1; echo rc=$?
grep k2_device gpurun_out/r2bi_repeat.jsonl | cut -c1-220
