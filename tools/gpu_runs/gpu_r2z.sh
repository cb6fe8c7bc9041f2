# round 2: 16-warp query_cta as the small-batch default (<= 16384 pairs): parity + sweep
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_reference_suites.py -q -m gpu -x > gpurun_out/r2z_parity.log 2>&1; echo parity_rc=$?
tail -2 gpurun_out/r2z_parity.log
timeout 900 python tools/query_sweep.py --config delaunay1m_k1024 --sizes 1e3,1e4,1.6e4,3e4,1e5,1e6 > gpurun_out/r2z_sweep.jsonl 2> gpurun_out/r2z_sweep.err; echo rc=$?
python -c "
import json
for l in open('gpurun_out/r2z_sweep.jsonl'):
    d=json.loads(l); print(d['batch_per_gpu'], d['kernel'], round(d['queries_per_s']/1e6,1), round((d.get('e2e_queries_per_s') or 0)/1e6,1))"
