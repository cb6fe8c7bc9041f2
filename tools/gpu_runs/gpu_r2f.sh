# round 2: PCIe ping-pong floor, point-query latency, acceptance
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
./tools/pcie_probe | tee gpurun_out/r2f_pcie.json
for args in "44 44 200000" "44 1 200000" "256 256 50000"; do
  PSP_SERVER_PROFILE=1 timeout 300 ./tools/latency_probe $args 2>&1
done | tee gpurun_out/r2f_latency.log
timeout 600 python -m pytest tests -q -m gpu -x -k "point_query or kernels_bitwise or large_boundaries" 2>&1 | tail -2
timeout 900 ./oracle/_ref/shim/gpu_acceptance > gpurun_out/r2f_acceptance.log 2>&1; echo acc_rc=$?
cat gpurun_out/r2f_acceptance.log
