# round 2: closing GPU suite + smoke at HEAD (f32 FW unroll 2)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/r2bm_pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/r2bm_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
grep '"config": "road4m' gpurun_out/large_configs.jsonl | cut -c1-300
