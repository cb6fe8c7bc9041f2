"""Multi-GPU build check (run under torchrun, one process per GPU).

Every rank builds the same oracle with the boundary-graph Floyd-Warshall
row-sharded over all ranks (NCCL), then checks it bit for bit against
(a) the committed reference fixture for BASELINE configs[0] and (b) a
single-GPU build of a Delaunay graph on the same device, and answers a
shard of queries. Prints one line per rank; exit code != 0 on mismatch.
"""
import hashlib
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1503_07192_b200 as P  # noqa: E402
from paper_1503_07192_b200 import graphs  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    dist.init_process_group("gloo")
    obj = [P.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    ctx = P.Context(local, rank, world, obj[0])
    solo = P.Context(local)

    z = np.load(os.path.join(ROOT, "tests", "golden", "ref_cfg1.npz"))
    g = P.Graph(int(z["n"]), z["eu"], z["ev"], z["ew"])
    o = P.build_oracle(g, 16, 4, 0, ctx=ctx)
    h = hashlib.sha256()
    for c in range(16):
        h.update(o.component_table(c).tobytes())
        h.update(o.boundary_rows(c).tobytes())
    ok = h.digest() == z["tables_sha256"].tobytes()
    d = o.batch_query(z["q_v1"], z["q_v2"])
    ok &= bool(np.array_equal(d, z["q_dist"]))

    # tiny boundary graphs: fewer tile rows than ranks (ranks with no rows)
    for rows, cols, k in ((2, 3, 2), (8, 8, 4), (20, 20, 9)):
        gt = P.generate_grid(rows, cols, (1, 9), rows)
        ot = P.build_oracle(gt, k, 2, 0, ctx=ctx)
        st = P.build_oracle(gt, k, 2, 0, ctx=solo)
        for c in range(k):
            ok &= bool(np.array_equal(ot.component_table(c), st.component_table(c)))
            ok &= bool(np.array_equal(ot.boundary_rows(c), st.boundary_rows(c)))

    gd = graphs.delaunay(30_000, 3)
    od = P.build_oracle(gd, 173, 4, 0, ctx=ctx)
    os_ = P.build_oracle(gd, 173, 4, 0, ctx=solo)
    for c in range(0, 173, 7):
        ok &= bool(np.array_equal(od.boundary_rows(c), os_.boundary_rows(c)))
    v1, v2 = P.random_pairs(gd.n, 200_000, 10 + rank)
    ok &= bool(np.array_equal(od.batch_query(v1, v2), os_.batch_query(v1, v2)))
    print(f"rank {rank}/{world}: cfg1 + delaunay30k sharded build "
          f"{'bit-exact' if ok else 'MISMATCH'} (k2 {od.stats['k2_device_ms']:.1f} ms sharded vs "
          f"{os_.stats['k2_device_ms']:.1f} ms single)", flush=True)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
