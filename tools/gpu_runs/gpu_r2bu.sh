# round 2: partitioner A/B after the parallel recenter (16-core GPU box): serial vs par on the last 2/4/8 chains; then bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python - <<'PY'
import sys, numpy as np
sys.path.insert(0, '.')
from paper_1503_07192_b200 import graphs
g, cfg = graphs.make("delaunay1m_k1024")
with open('/tmp/cfg3.bin', 'wb') as f:
    np.array([g.n, len(g.eu)], np.uint64).tofile(f)
    g.eu.astype(np.uint32).tofile(f); g.ev.astype(np.uint32).tofile(f); g.ew.astype(np.float64).tofile(f)
PY
nproc
for i in 1 2; do
echo -n "serial "; PSP_PART_SERIAL=1 ./tools/part_bench /tmp/cfg3.bin 1024 16 1 2>&1 | grep hash
for L in 2 4 6 8; do
echo -n "last=$L "; PSP_PART_PAR_LAST=$L ./tools/part_bench /tmp/cfg3.bin 1024 16 1 2>&1 | grep hash
done; done
PSP_PART_PROFILE=1 ./tools/part_bench /tmp/cfg3.bin 1024 16 1 2>&1 | tail -14
timeout 1500 python bench.py --no-cpu-baseline > gpurun_out/r2bu_bench.json 2> gpurun_out/r2bu_bench.err; echo bench_rc=$?
python -c "import json;d=json.load(open('gpurun_out/r2bu_bench.json'));p=d['preprocessing'];print(d['value'], d['e2e']['value'], p['partition_s'], p['preprocessing_s'])"
