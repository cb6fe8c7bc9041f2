# round 2: point-query latency path + acceptance through the shim
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -s -k "point_query or kernels_bitwise or large_boundaries or registry or concurrent" > gpurun_out/r2c_pytest.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/r2c_pytest.log; grep "point query" gpurun_out/r2c_pytest.log
timeout 900 ./oracle/_ref/shim/gpu_acceptance > gpurun_out/r2c_acceptance.log 2>&1; echo acc_rc=$?
cat gpurun_out/r2c_acceptance.log
