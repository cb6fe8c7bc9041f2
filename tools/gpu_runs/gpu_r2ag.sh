# round 2: launch list of the bench's timed query steps (ncu profiles only the query-step kernels)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name regex:'group|query|minplus' --csv --log-file gpurun_out/r2ag_launches_query_steps.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2ag_ncu_bench.log 2>&1; echo ncu_rc=$?
python tools/launch_summary.py gpurun_out/r2ag_launches_query_steps.csv 2>&1 | tail -20
