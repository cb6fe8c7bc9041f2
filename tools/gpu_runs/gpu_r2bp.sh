# round 2: partitioner with parallel grows on the last two chains vs serial (16-core GPU box)
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
for i in 1 2; do
PSP_PART_SERIAL=1 PSP_PART_PROFILE=1 ./tools/part_bench /tmp/cfg3.bin 1024 16 1 2>&1 | grep "chain 7\|hash" | tr '\n' ' '; echo serial
PSP_PART_PROFILE=1 ./tools/part_bench /tmp/cfg3.bin 1024 16 1 2>&1 | grep "chain 7\|hash" | tr '\n' ' '; echo par
done
