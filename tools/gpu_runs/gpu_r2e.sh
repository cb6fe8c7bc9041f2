# round 2: point-query latency breakdown, PSP1 file throughput, small-batch kernel sweep
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for args in "44 44 200000" "44 1 200000" "20 4 200000" "256 256 50000"; do
  PSP_SERVER_PROFILE=1 timeout 300 ./tools/latency_probe $args 2>&1
done | tee gpurun_out/r2e_latency.log
timeout 600 python -m pytest tests/test_gpu_oracle_file.py -q -x 2>&1 | tail -2
timeout 900 python tools/file_bench.py --config delaunay262k_k256 2>&1 | tail -2 | tee gpurun_out/r2e_file.log
timeout 1200 python tools/query_sweep.py --config delaunay1m_k1024 --sizes 1e3,1e4,3e4,1e5,3e5,1e6,1e7 --kernels cta,grouped --no-e2e > gpurun_out/r2e_sweep.jsonl 2> gpurun_out/r2e_sweep.err; echo sweep_rc=$?
cat gpurun_out/r2e_sweep.jsonl; tail -3 gpurun_out/r2e_sweep.err
