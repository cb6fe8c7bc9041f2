# round 2: cfg3 boundary-phase laps over 4 repeated builds (PSP_FW_PROFILE)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
PSP_FW_PROFILE=1 timeout 900 python tools/build_repeat.py --config delaunay1m_k1024 --builds 4 > gpurun_out/r2aa_repeat.jsonl 2> gpurun_out/r2aa_repeat.err; echo rc=$?
grep "boundary lap\|K2 permutation\|component phase\|order chosen" gpurun_out/r2aa_repeat.err | cut -c1-160
cat gpurun_out/r2aa_repeat.jsonl
