# round 2: GPU suite (incl. acceptance through the shim), cfg3 bench both arms
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -s -k "point_query or concurrent or kernels_bitwise or large_boundaries or registry or acceptance" > gpurun_out/r2b_pytest_new.log 2>&1; echo pytest_new_rc=$?
tail -5 gpurun_out/r2b_pytest_new.log
grep -E "criterion|point query" gpurun_out/r2b_pytest_new.log | head -20
timeout 1200 python bench.py > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err; echo bench_rc=$?
tail -c 3000 gpurun_out/r2b_bench.json; tail -5 gpurun_out/r2b_bench.err
timeout 1500 python bench.py --impl reference > gpurun_out/r2b_ref.json 2> gpurun_out/r2b_ref.err; echo ref_rc=$?
tail -c 2500 gpurun_out/r2b_ref.json; tail -5 gpurun_out/r2b_ref.err
