# round 2: partitioner A/B on the 16-core GPU box after keeping the winner's finalized state:
# serial chains vs parallel grows (+/- parallel recenter) on the last 2/4 chains, 4 interleaved reps
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
for i in 1 2 3 4; do
echo -n "serial "; PSP_PART_SERIAL=1 ./tools/part_bench /tmp/cfg3.bin 1024 16 1 2>&1 | grep hash
for L in 2 4; do
echo -n "last=$L "; PSP_PART_PAR_LAST=$L ./tools/part_bench /tmp/cfg3.bin 1024 16 1 2>&1 | grep hash
echo -n "last=$L serial-recenter "; PSP_PART_SERIAL_RECENTER=1 PSP_PART_PAR_LAST=$L ./tools/part_bench /tmp/cfg3.bin 1024 16 1 2>&1 | grep hash
done; done
