"""Multi-GPU routed-query check (run under torchrun, one process per GPU).

Every rank builds the replicated oracle (boundary-graph FW row-sharded over
the ranks), then a RoutedOracle per placement policy keeps only its own
components' tables and answers batches at owner(C1), reading col2 from
owner(C2)'s GPU over NVLink. Checks, per policy:
  A. rank 0 submits the first 4000 configs[0] fixture pairs, the others
     none: distances and the transfer ledger equal the reference
     ClusterSim's (tests/golden/ref_cluster_cfg1.npz, p = world);
  B. every rank submits its own random pairs on a 30k-vertex Delaunay graph:
     distances bit-equal to the replicated oracle's batch_query;
  C. an out-of-range id on the last rank fails the batch on every rank;
  D. row-sharded storage (STORAGE_ROW_SHARDED): the same graphs built with
     only each rank's tile rows of the boundary-graph table on its GPU (the
     Delaunay one also with the tile-packed K2 layout forced); replicated
     queries are refused and RoutedOracle answers A's and B's pairs bit-equal
     to the replicated oracle. (Tables this small fit in a few 2 MB granules,
     so the memory share is checked at full size: tools/row_storage_check.py.)
Prints "routed_check: ok" on rank 0 when every rank passed.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("NCCL_DEBUG", "WARN")
import paper_1503_07192_b200 as P  # noqa: E402
from paper_1503_07192_b200 import graphs  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    dist.init_process_group("gloo")
    obj = [P.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    ctx = P.Context(local, rank, world, obj[0])
    fails = []

    z = np.load(os.path.join(ROOT, "tests", "golden", "ref_cfg1.npz"))
    zc = np.load(os.path.join(ROOT, "tests", "golden", "ref_cluster_cfg1.npz"))
    g = P.Graph(int(z["n"]), z["eu"], z["ev"], z["ew"])
    o = P.build_oracle(g, 16, 4, 0, ctx=ctx)
    gd = graphs.delaunay(30_000, 3)
    od = P.build_oracle(gd, 173, 4, 0, ctx=ctx)
    v1, v2 = P.random_pairs(gd.n, 300_000, 20 + rank)
    want_d = od.batch_query(v1, v2)

    for pol_i, policy in ((0, P.ROUND_ROBIN), (1, P.PAIRS_PER_GPU)):
        # A: reference ClusterSim ledger (fixture made for p = 2 and 4)
        key = f"p{world}_pol{pol_i}"
        ro = P.RoutedOracle(o, P.place_components(16, world, policy))
        mine = (zc["v1"], zc["v2"]) if rank == 0 else (np.empty(0, np.uint32),) * 2
        d = ro.run_batch(*mine)
        if rank == 0 and f"{key}_ledger" in zc:
            if not np.array_equal(d, zc[f"{key}_dist"]):
                fails.append(f"A/{policy}: distances differ from ClusterSim")
            got = np.array([[r.query_id, r.src_worker, r.dst_worker, r.entries, r.bytes]
                            for r in ro.ledger().records()], np.uint64).reshape(-1, 5)
            if not np.array_equal(got, zc[f"{key}_ledger"]):
                fails.append(f"A/{policy}: ledger differs ({len(got)} vs {len(zc[key + '_ledger'])})")
            st = ro.last_stats
            if st["transfer_bytes"] != ro.ledger().total_bytes():
                fails.append(f"A/{policy}: stats bytes {st['transfer_bytes']} != ledger")
        ro.close()

        # B: every rank its own batch on the Delaunay oracle
        rd = P.RoutedOracle(od, P.place_components(173, world, policy))
        got, ex, co, ent = rd.run_batch(v1, v2, with_routing=True)
        if not np.array_equal(got, want_d):
            bad = np.nonzero(got != want_d)[0]
            fails.append(f"B/{policy}: {len(bad)} distances differ, first {bad[:3]}")
        pl = rd.placement
        c1 = od.assignment[od.permutation[v1.astype(np.int64)]]
        c2 = od.assignment[od.permutation[v2.astype(np.int64)]]
        if not (np.array_equal(ex, pl.owner[c1]) and np.array_equal(co, pl.owner[c2])):
            fails.append(f"B/{policy}: routing facts differ")
        st = rd.last_stats
        print(f"rank {rank}/{world} {policy}: {len(v1)} pairs, executed here {st['executed_here']}, "
              f"sent {st['sent_to_peers']}, col2 over NVLink {st['transfer_queries']} "
              f"({st['transfer_entries']} entries), route {st['route_ms']:.2f} ms, "
              f"exec {st['exec_ms']:.2f} ms, shard {rd.device_bytes() / 1e6:.1f} MB", flush=True)

        # C: a bad id anywhere fails everywhere
        bad1 = v1[:100].copy()
        if rank == world - 1:
            bad1[7] = gd.n
        try:
            rd.run_batch(bad1, v2[:100])
            fails.append(f"C/{policy}: bad id not reported")
        except ValueError:
            pass
        rd.close()

    # D: row-sharded boundary-graph storage
    ctx.set_boundary_storage(P.STORAGE_ROW_SHARDED)
    want_a = o.batch_query(zc["v1"], zc["v2"])
    rep_bytes = od.stats["device_bytes"]
    for force_pack in (False, True):
        if force_pack:
            os.environ["PSP_BG_PACK"] = "force"
        os_ = P.build_oracle(g, 16, 4, 0, ctx=ctx)
        ods = P.build_oracle(gd, 173, 4, 0, ctx=ctx)
        os.environ.pop("PSP_BG_PACK", None)
        tag = "D/packed" if force_pack else "D"
        try:
            ods.batch_query(v1[:10], v2[:10])
            fails.append(f"{tag}: replicated query on a row-sharded oracle not refused")
        except ValueError:
            pass
        st = ods.stats
        nb = (st["k2_positions"] + 127) // 128
        table = nb * (nb + 1) // 2 * 128 * 128 * 4
        rows = range(rank, nb, world)
        mine_bytes = sum((nb - I) * 128 * 128 * 4 for I in rows)
        print(f"rank {rank}/{world} {tag}: table {table / 1e6:.1f} MB, owned rows {mine_bytes / 1e6:.1f} MB, "
              f"oracle device bytes {st['device_bytes'] / 1e6:.1f} MB (replicated {rep_bytes / 1e6:.1f} MB), "
              f"k2 positions {st['k2_positions']} order {st['k2_order']}", flush=True)
        if force_pack and not (st["k2_order"] == 1 and st["k2_positions"] > ods.b):
            fails.append(f"{tag}: tile-packed layout not taken ({st['k2_positions']} positions)")
        for pol_i, policy in ((0, P.ROUND_ROBIN), (1, P.PAIRS_PER_GPU)):
            ro = P.RoutedOracle(os_, P.place_components(16, world, policy))
            mine = (zc["v1"], zc["v2"]) if rank == 0 else (np.empty(0, np.uint32),) * 2
            d = ro.run_batch(*mine)
            if rank == 0 and not np.array_equal(d, want_a):
                fails.append(f"{tag}/A/{policy}: distances differ from the replicated oracle")
            ro.close()
            rd = P.RoutedOracle(ods, P.place_components(173, world, policy))
            got = rd.run_batch(v1, v2)
            if not np.array_equal(got, want_d):
                bad = np.nonzero(got != want_d)[0]
                fails.append(f"{tag}/B/{policy}: {len(bad)} distances differ, first {bad[:3]}")
            rd.close()
        os_.close()
        ods.close()
    ctx.set_boundary_storage(P.STORAGE_REPLICATED)

    ok = torch.tensor([0 if fails else 1])
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    for f in fails:
        print(f"rank {rank}: FAIL {f}", flush=True)
    if rank == 0 and ok.item():
        print("routed_check: ok", flush=True)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok.item() else 1)


if __name__ == "__main__":
    main()
