# round 2: partitioner A/B on configs[3] (road4m, k=512) on the 16-core GPU box: timeline + serial / last 2 / 4 / 8
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python - <<'PY'
import sys, numpy as np
sys.path.insert(0, '.')
from paper_1503_07192_b200 import graphs
g, cfg = graphs.make("road4m_k512")
with open('/tmp/road4m.bin', 'wb') as f:
    np.array([g.n, len(g.eu)], np.uint64).tofile(f)
    g.eu.astype(np.uint32).tofile(f); g.ev.astype(np.uint32).tofile(f); g.ew.astype(np.float64).tofile(f)
PY
PSP_PART_PROFILE=1 ./tools/part_bench /tmp/road4m.bin 512 16 1 2>&1 | tail -16
for i in 1 2; do
echo -n "serial "; PSP_PART_SERIAL=1 ./tools/part_bench /tmp/road4m.bin 512 16 1 2>&1 | grep hash
for L in 2 4 8; do
echo -n "last=$L "; PSP_PART_PAR_LAST=$L ./tools/part_bench /tmp/road4m.bin 512 16 1 2>&1 | grep hash
done; done
