"""Row-sharded boundary-graph storage at full size (run under torchrun, one
process per GPU).

Every rank builds a BASELINE configuration with STORAGE_ROW_SHARDED: the
row-sharded K2 keeps only the tile rows this rank computed, so the boundary
table's per-rank share is ~1/world and a table larger than one GPU can be
built across several. Then RoutedOracle (round-robin placement) gathers each
rank's components' boundary rows from the distributed rows (ncclReduce) and
answers routed queries. Checks:
  * per rank, the table bytes held (oracle device bytes minus the replicated
    component / to-boundary tables) against table / world;
  * rank 0 submits SOURCES x TARGETS pairs, the others none: distances bit-equal
    (u32) to f64 Dijkstra on the original graph (oracle/psp_oracle.c, the
    reference's cmd_verify pattern, proj/tools/psp_main.cpp:237-283);
  * every rank submits BATCH random pairs: the routed throughput.
Rank 0 prints one JSON line and "row_storage_check: ok" when every rank passed.

  torchrun --standalone --nproc-per-node 2 tools/row_storage_check.py --config delaunay1m_k1024
"""
import argparse
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("NCCL_DEBUG", "WARN")
import oracle  # noqa: E402  (test-side checker only: Dijkstra)
import paper_1503_07192_b200 as P  # noqa: E402
from paper_1503_07192_b200 import graphs  # noqa: E402

SOURCES, TARGETS = 16, 20_000


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="delaunay262k_k256")
    ap.add_argument("--batch", type=int, default=2_000_000)
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    dist.init_process_group("gloo")
    obj = [P.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    ctx = P.Context(local, rank, world, obj[0])
    ctx.set_boundary_storage(P.STORAGE_ROW_SHARDED)
    fails = []

    g, cfg = graphs.make(args.config)
    t0 = time.time()
    o = P.build_oracle(g, cfg["k"], os.cpu_count() or 8, 0, ctx=ctx)
    build_s = time.time() - t0
    st = o.stats
    exact = o.value_kind == P.VALUE_U32
    vb = 4
    nb = (st["k2_positions"] + 127) // 128
    table = nb * (nb + 1) // 2 * 128 * 128 * vb
    owned = sum((nb - I) * 128 * 128 * vb for I in range(rank, nb, world))
    try:
        o.batch_query(np.zeros(1, np.uint32), np.zeros(1, np.uint32))
        fails.append("replicated query on a row-sharded oracle not refused")
    except ValueError:
        pass

    t0 = time.time()
    ro = P.RoutedOracle(o, P.place_components(cfg["k"], world, P.ROUND_ROBIN))
    shard_s = time.time() - t0
    shard_bytes = ro.device_bytes()
    oracle_bytes = st["device_bytes"]
    o.close()  # the distributed rows are no longer needed

    # exactness: rank 0's pairs vs Dijkstra
    rng = np.random.default_rng(5)
    sources = rng.choice(g.n, size=SOURCES, replace=False)
    targets = rng.choice(g.n, size=TARGETS, replace=False).astype(np.uint32)
    if rank == 0:
        v1 = np.repeat(sources.astype(np.uint32), TARGETS)
        v2 = np.tile(targets, SOURCES)
    else:
        v1 = v2 = np.empty(0, np.uint32)
    d = ro.run_batch(v1, v2)
    mismatches = max_rel = 0
    if rank == 0:
        off, to, w = oracle.csr(g.n, g.eu, g.ev, g.ew)
        lib = oracle.Oracle.lib()

        def truth_row(s):
            t = np.empty(g.n)
            lib.pso_dijkstra(g.n, off, to, w, int(s), t)
            return t[targets]

        with ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 4)) as ex:
            t = np.concatenate(list(ex.map(truth_row, sources)))
        if exact:
            mismatches = int((d != t).sum())
        else:
            rel = np.abs(d - t) / np.maximum(t, 1e-300)
            max_rel = float(rel.max())
            mismatches = int((rel > 1e-5).sum())
        if mismatches:
            fails.append(f"{mismatches} of {len(t)} distances differ from Dijkstra")

    # routed throughput: every rank its own batch
    a1, a2 = P.random_pairs(g.n, args.batch, 100 + rank)
    ro.run_batch(a1, a2)  # warm-up
    dist.barrier()
    t0 = time.time()
    reps = 3
    for _ in range(reps):
        ro.run_batch(a1, a2)
    dist.barrier()
    wall = (time.time() - t0) / reps
    ls = ro.last_stats
    ro.close()

    info = torch.tensor([owned, oracle_bytes, shard_bytes, int(build_s * 1e3), int(shard_s * 1e3),
                         int(wall * 1e6)], dtype=torch.int64)
    gathered = [torch.zeros_like(info) for _ in range(world)]
    dist.all_gather(gathered, info)
    okt = torch.tensor([0 if fails else 1])
    dist.all_reduce(okt, op=dist.ReduceOp.MIN)
    for f in fails:
        print(f"rank {rank}: FAIL {f}", flush=True)
    if rank == 0:
        per = [x.tolist() for x in gathered]
        line = {"config": args.config, "world": world, "n": g.n, "k": cfg["k"], "b": o.b,
                "value_kind": "u32" if exact else "f32", "table_bytes": table,
                "owned_row_bytes_per_rank": [p[0] for p in per],
                "oracle_device_bytes_per_rank": [p[1] for p in per],
                "shard_device_bytes_per_rank": [p[2] for p in per],
                "build_s": [p[3] / 1e3 for p in per], "shard_create_s": [p[4] / 1e3 for p in per],
                "k2_device_s": round(st["k2_device_ms"] / 1e3, 3),
                "k2_positions": st["k2_positions"], "k2_order": st["k2_order"],
                "pairs_checked_vs_dijkstra": SOURCES * TARGETS, "mismatches": mismatches,
                "max_rel_err": max_rel,
                "routed_batch_per_rank": args.batch,
                "routed_queries_per_s": world * args.batch / (max(p[5] for p in per) / 1e6),
                "routed_last_stats_rank0": ls}
        print(json.dumps(line), flush=True)
        os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
        with open(os.path.join(ROOT, "gpurun_out", "row_storage.jsonl"), "a") as f:
            f.write(json.dumps(line) + "\n")
        if okt.item():
            print("row_storage_check: ok", flush=True)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if okt.item() else 1)


if __name__ == "__main__":
    main()
