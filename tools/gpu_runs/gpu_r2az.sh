# round 2: allocation cost probe (cudaMalloc vs VMM create/map, first touch)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 ./tools/alloc_probe2 > gpurun_out/r2az_alloc.log 2>&1; echo rc=$?
cat gpurun_out/r2az_alloc.log
