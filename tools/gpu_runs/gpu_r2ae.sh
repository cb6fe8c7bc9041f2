# round 2: streamed PSP1 load (device CRC + conversion): file tests + cfg2 save/load timing
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_oracle_file.py -q -m gpu -x > gpurun_out/r2ae_file.log 2>&1; echo file_rc=$?
tail -2 gpurun_out/r2ae_file.log
timeout 1200 python tools/file_bench.py --config delaunay262k_k256 > gpurun_out/r2ae_psp1_cfg2.json 2> gpurun_out/r2ae_psp1.err; echo bench_rc=$?
cat gpurun_out/r2ae_psp1_cfg2.json
