"""Routed (sharded-table) query throughput vs replicated tables, under
torchrun (one process per GPU).

Every rank builds the replicated oracle (BG FW row-sharded), then
  replicated: each rank answers its own batch from its full copy
              (psp_gpu_query_batch, host pairs in, distances out);
  routed:     RoutedOracle keeps only this rank's components (placement
              policy --policy); each rank submits its own batch, queries
              execute at owner(C1) with col2 read from owner(C2) over NVLink
              (psp_gpu_routed_query_batch, host pairs in, distances out).
Both are timed end to end per batch (host API, max over ranks). Prints one
JSON line on rank 0.

  torchrun --nproc-per-node 2 tools/routed_bench.py [--config delaunay262k_k256]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("NCCL_DEBUG", "WARN")
import paper_1503_07192_b200 as P  # noqa: E402
from paper_1503_07192_b200 import graphs  # noqa: E402


def timed(fn, reps):
    dist.barrier()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    el = torch.tensor([(time.perf_counter() - t) / reps], dtype=torch.float64)
    dist.all_reduce(el, op=dist.ReduceOp.MAX)
    return float(el.item())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="delaunay262k_k256")
    ap.add_argument("--batch", type=int, default=1_000_000, help="pairs per rank per batch")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--policy", default=P.ROUND_ROBIN, choices=[P.ROUND_ROBIN, P.PAIRS_PER_GPU])
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    dist.init_process_group("gloo")
    obj = [P.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    ctx = P.Context(local, rank, world, obj[0])
    g, cfg = graphs.make(args.config)
    part = [P.partition_graph(g, cfg["k"], 0, os.cpu_count()) if rank == 0 else None]
    dist.broadcast_object_list(part, src=0)
    o = P.build_partitioned(g, cfg["k"], part[0], ctx=ctx)
    v1, v2 = P.random_pairs(g.n, args.batch, 700 + rank)
    for _ in range(3):
        want = o.batch_query(v1, v2)
    rep_s = timed(lambda: o.batch_query(v1, v2), args.reps)
    full_bytes = int(o.stats["device_bytes"])

    pl = P.place_components(o.k, world, args.policy)
    ro = P.RoutedOracle(o, pl)
    o.close()  # this rank now holds only its own components' tables
    torch.cuda.synchronize(local)
    for _ in range(3):
        got = ro.run_batch(v1, v2)
    ok = bool(np.array_equal(got, want))
    routed_s = timed(lambda: ro.run_batch(v1, v2), args.reps)
    st = ro.last_stats
    res = torch.tensor([st["route_ms"], st["exec_ms"], ro.device_bytes(), 0 if ok else 1],
                       dtype=torch.float64)
    dist.all_reduce(res, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({
            "config": args.config, "n_gpus": world, "policy": args.policy,
            "batch_per_rank": args.batch,
            "replicated_e2e_queries_per_s": round(args.batch * world / rep_s, 1),
            "routed_e2e_queries_per_s": round(args.batch * world / routed_s, 1),
            "routed_route_ms_max": round(res[0].item(), 3),
            "routed_exec_ms_max": round(res[1].item(), 3),
            "transfer_queries_rank0": st["transfer_queries"],
            "transfer_bytes_rank0_f64_ledger": st["transfer_bytes"],
            "replicated_device_bytes_per_gpu": full_bytes,
            "routed_device_bytes_per_gpu_max": int(res[2].item()),
            "bit_exact": res[3].item() == 0,
        }), flush=True)
    ro.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
