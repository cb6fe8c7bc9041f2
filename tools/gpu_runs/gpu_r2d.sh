# round 2: point-query server with smem-cached ids; DPX u16x2 probe
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
./tools/minplus_probe > gpurun_out/r2d_minplus_probe.json 2>&1; cat gpurun_out/r2d_minplus_probe.json
timeout 900 python -m pytest tests -q -m gpu -s -k "point_query or registry" > gpurun_out/r2d_pytest.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/r2d_pytest.log; grep "point query" gpurun_out/r2d_pytest.log
timeout 900 ./oracle/_ref/shim/gpu_acceptance > gpurun_out/r2d_acceptance.log 2>&1; echo acc_rc=$?
cat gpurun_out/r2d_acceptance.log
