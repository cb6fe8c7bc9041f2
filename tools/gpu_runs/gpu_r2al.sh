# round 2: blocking host API through pinned staging (<= 1M pairs): parity + small-batch e2e sweep
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_reference_suites.py -q -m gpu -x > gpurun_out/r2al_parity.log 2>&1; echo parity_rc=$?
tail -1 gpurun_out/r2al_parity.log
timeout 900 python tools/query_sweep.py --config delaunay1m_k1024 --sizes 1e3,1e4,1e5,1e6 > gpurun_out/r2al_sweep.jsonl 2> gpurun_out/r2al_sweep.err; echo rc=$?
python -c "
import json
for l in open('gpurun_out/r2al_sweep.jsonl'):
    d=json.loads(l); print(d['batch_per_gpu'], d['kernel'], round(d['queries_per_s']/1e6,1), round((d.get('e2e_queries_per_s') or 0)/1e6,1))"
