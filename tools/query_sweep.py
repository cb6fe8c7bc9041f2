"""BASELINE.json configs[4]: query-throughput sweep, batch sizes 1K..100M of
random pairs on the 1M-vertex Delaunay structure, at N GPUs (run under
torchrun for N > 1; queries sharded by rank, tables built with the
row-sharded boundary-graph FW).

For every batch size: device-resident queries/s (pairs already in HBM, CUDA
events, max over ranks) and end-to-end queries/s through psp_gpu_query_batch
(pinned host pairs, H2D + D2H inside the timed region). Dense batches run
query_grouped, sparse ones query_warp (the library picks by density).
Prints one JSON line per batch size on rank 0.

  python tools/query_sweep.py [--config delaunay1m_k1024] [--sizes 1e3,1e4,...]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("NCCL_DEBUG", "WARN")

import paper_1503_07192_b200 as P  # noqa: E402
from paper_1503_07192_b200 import graphs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="delaunay1m_k1024")
    ap.add_argument("--sizes", default="1e3,1e4,1e5,1e6,1e7,1e8")
    ap.add_argument("--min-time", type=float, default=0.25, help="seconds per measurement")
    ap.add_argument("--kernels", default="auto",
                    help="comma list of auto|warp|grouped|cta: force a query kernel "
                         "(PSP_QUERY_KERNEL) instead of the density rule, each measured")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        obj = [P.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ctx = P.Context(local, rank, world, obj[0])
    else:
        ctx = P.Context(local)
    g, cfg = graphs.make(args.config)
    t0 = time.time()
    if world > 1:
        part = torch.empty(g.n, dtype=torch.int32, device=dev)
        if rank == 0:
            part.copy_(torch.from_numpy(P.partition_graph(g, cfg["k"], 0, os.cpu_count()).view(np.int32)))
        dist.broadcast(part, src=0)
        o = P.build_partitioned(g, cfg["k"], part.cpu().numpy().view(np.uint32), ctx=ctx)
    else:
        o = P.build_oracle(g, cfg["k"], os.cpu_count(), 0, ctx=ctx)
    build_s = time.time() - t0
    stream = torch.cuda.Stream(device=dev)
    lib = P._lib.lib()
    for size, kernel in [(int(float(x)), kname) for x in args.sizes.split(",")
                         for kname in args.kernels.split(",")]:
        if kernel == "auto":
            os.environ.pop("PSP_QUERY_KERNEL", None)
        else:
            os.environ["PSP_QUERY_KERNEL"] = kernel
        v1, v2 = P.random_pairs(g.n, size, 500 + rank)
        d1 = torch.from_numpy(v1.view(np.int32)).to(dev)
        d2 = torch.from_numpy(v2.view(np.int32)).to(dev)
        out = torch.empty(size, dtype=torch.float64, device=dev)

        def step():
            o.batch_query_device(d1.data_ptr(), d2.data_ptr(), out.data_ptr(), size,
                                 stream.cuda_stream)

        for _ in range(3):
            step()
        torch.cuda.synchronize()
        # repetitions so the measurement spans >= min_time
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)
        torch.cuda.synchronize()
        reps = max(1, int(args.min_time / max(e0.elapsed_time(e1) / 1e3, 1e-6)))
        if dist:
            r = torch.tensor([reps], device=dev)
            dist.all_reduce(r, op=dist.ReduceOp.MAX)
            reps = int(r.item())
            dist.barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(reps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        dev_s = e0.elapsed_time(e1) / 1e3 / reps
        h1 = torch.from_numpy(v1.view(np.int32)).pin_memory()
        h2 = torch.from_numpy(v2.view(np.int32)).pin_memory()
        ho = torch.empty(size, dtype=torch.float64).pin_memory()

        def e2e():
            P._lib.check(lib.psp_gpu_query_batch(o.h, size, h1.data_ptr(), h2.data_ptr(),
                                                 ho.data_ptr(), None))

        e2e_s = float("nan")
        if not args.no_e2e:
            for _ in range(3):
                e2e()
            if dist:
                dist.barrier()
            t = time.perf_counter()
            for _ in range(reps):
                e2e()
            e2e_s = (time.perf_counter() - t) / reps
        times = torch.tensor([dev_s, e2e_s], dtype=torch.float64, device=dev)
        if dist:
            dist.all_reduce(times, op=dist.ReduceOp.MAX)
        dev_s, e2e_s = times.tolist()
        pairs = o.k * (o.k + 1) / 2
        used = kernel if kernel != "auto" else (
            "cta" if size < P.CTA_MAX_DENSITY * pairs or size <= P.CTA_MAX_COUNT else "grouped")
        if used == "grouped":
            used += (" (sparse grouping)" if o.k * o.k >= P.SPARSE_GROUPING_MIN_BINS
                     and size * P.SPARSE_GROUPING_RATIO < o.k * o.k else "")
        if rank == 0:
            print(json.dumps({"config": args.config, "n_gpus": world, "batch_per_gpu": size,
                              "kernel": "query_" + used, "forced": kernel != "auto",
                              "queries_per_s": round(size * world / dev_s, 1),
                              "e2e_queries_per_s": round(size * world / e2e_s, 1),
                              "ms_per_batch": round(dev_s * 1e3, 4), "reps": reps,
                              "build_s": round(build_s, 2)}), flush=True)
        del d1, d2, out, h1, h2, ho
        torch.cuda.empty_cache()
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
