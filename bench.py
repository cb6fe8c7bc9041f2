#!/usr/bin/env python
"""Benchmark: distance queries/s (+ preprocessing seconds) on B200.

Contract:
  python bench.py --gpus N --steps K --warmup W [--impl ours|reference]
Under torchrun (N > 1) each rank drives one GPU; rank 0 prints ONE JSON line.

Workload: BASELINE.json configs[2], the configuration the metric is quoted on
("1M-vertex planar"), which fits one B200: Delaunay triangulation of
1,048,576 uniform points, integer weights 1..1024, k = 1024 components
(b = 135,009), batches of 10,000,000 random pairs per step per GPU. Every
rank builds the oracle (partition on the host, phases 2-3 on the GPUs, the
boundary-graph FW row-sharded over the ranks) and answers its own batches
("scaling": "weak", queries sharded by rank, no data-path collective: the
query path needs none when every GPU holds the tables).
`--config delaunay262k_k256` gives the configs[1] line.

value  device-resident queries/s over all ranks (pairs already in HBM,
       CUDA events on the launching stream, max over ranks)
e2e    the same batches through the pipelined host API with pinned host
       pairs: H2D of 8 B/pair and D2H of 8 B/distance inside the timed region
Inputs (the 36.5 GB boundary-graph table) are far larger than the 126 MB L2,
so no flush is needed between steps; each step uses a fresh slice of pairs.

--impl reference runs the UNMODIFIED reference (oracle/_ref/libpspref.so,
built from /root/reference/proj/src by oracle/Makefile) on the host cores and
never imports the product package (workloads.py draws the graph). Where the
reference's f64 boundary tables exceed host RAM (cfg3: 145.8 GB) its Phase 3
runs on a seeded sample of components (labelled
"extrapolated") and its queries start in those components.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# rank 0 must print exactly one JSON line on stdout: keep NCCL's version
# banner off stdout unless the caller asked for NCCL logging
os.environ.setdefault("NCCL_DEBUG", "WARN")

FAMILY = {"grid": "grid", "delaunay": "Delaunay", "road": "road-like grid (f32 weights)"}
METRIC = "distance queries/sec + preprocessing s (1M-vertex planar) at 1/2/4/8 B200 vs CPU"
CONFIG = "delaunay1m_k1024"
# components whose boundary rows the reference computes where its full
# f64 tables exceed host RAM
REF_COMPONENTS = 16
# the reference builds in full up to this many vertices (cfg2: 9.8 GB of f64
# boundary tables), with a sampled Phase 3 beyond
REF_FULL_MAX_N = 300_000
BATCH = 1_000_000


def measured_peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        d["source"] = "measured (MEASURED_PEAKS.json)"
        return d
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    """SM clocks + throttle reasons sampled through NVML every ~10 ms during
    the timed region (the B200_PROFILING.md clocks line, in-process so that
    even a sub-second region gets many samples); falls back to nvidia-smi."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))

    def __init__(self, device: int, period_s: float = 0.01):
        self.device = device
        self.period = period_s
        self.sm, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._t = None
        self._nvml = None

    def _sample_nvml(self, h):
        nv = self._nvml
        self.sm.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
        mask = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        for name, attr in self.REASONS:
            if mask & getattr(nv, attr, 0):
                self.reasons.add(name)

    def _sample_smi(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True,
                             timeout=5)
        vals = [v.strip() for v in out.stdout.strip().split(",")]
        if len(vals) == 6:
            self.sm.append(float(vals[0]))
            self.max_mhz = float(vals[1])
            for i, (name, _) in enumerate(self.REASONS):
                if vals[2 + i].lower() == "active":
                    self.reasons.add(name)

    def _run(self):
        h = None
        try:
            import pynvml as nv
            nv.nvmlInit()
            self._nvml = nv
            h = nv.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        except Exception:
            self._nvml = None
        while True:
            try:
                if self._nvml is not None:
                    self._sample_nvml(h)
                else:
                    self._sample_smi()
            except Exception:
                pass
            if self._stop.wait(self.period if self._nvml is not None else 0.2):
                break

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self) -> dict:
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["no samples"],
                    "samples": 0}
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.sm),
                "source": "nvml" if self._nvml is not None else "nvidia-smi"}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def query_bytes_and_ops(o, v1, v2):
    """Algorithmic bytes / ops per query: 4(B1 B2 + B1 + B2) + 28
    bytes (u32 tables, no reuse; 8 B pair in, 4 B out, 16 B id lookups) and
    B1 B2 + B2 relaxations (the reference's minplus_ops, src/query.cpp:73)."""
    bsz = np.diff(o.boundary_offset).astype(np.float64)
    comp = o.assignment[o.permutation]
    b1 = bsz[comp[v1]]
    b2 = bsz[comp[v2]]
    byts = 4.0 * (b1 * b2 + b1 + b2) + 28.0
    ops = b1 * b2 + b2
    return float(byts.sum()), float(ops.sum())


def grouped_executed_relaxations(k, bsize, c1, c2):
    """Relaxations query_grouped EXECUTES for a batch (thread level, incl. the
    padding of its lane layout), from the task rules of group_tasks /
    group_emit and group_task_rb (query_kernels.cuh): pairs oriented c1 <= c2
    and binned; a bin's nq queries split into ceil(nq / 32) balanced items
    (mbig = min(32, ceil(nq / items) rounded up to 4)); per item and 32-column
    group, 4 * ceil(m / 4) query slots x 32 columns (the pair's last group, if
    it holds <= 16 columns: 8 * ceil(m / 8) slots x 16 columns) x the rows
    walked (16-row chunks, each rounded up to 4 rows) plus one pass for the
    col2 combine. `useful / executed` is the padding share of the ALU work."""
    a = np.minimum(c1, c2).astype(np.int64)
    b = np.maximum(c1, c2).astype(np.int64)
    keys, nq = np.unique(a * k + b, return_counts=True)
    B1 = bsize[keys // k].astype(np.int64)
    B2 = bsize[keys % k].astype(np.int64)
    items = (nq + 31) // 32
    mbig = np.minimum(32, ((nq + items - 1) // items + 3) // 4 * 4)
    m_last = nq - (items - 1) * mbig
    ncg = (B2 + 31) // 32
    half = (B2 - (ncg - 1) * 32) <= 16
    rows = 16 * (B1 // 16) + (B1 % 16 + 3) // 4 * 4 + 1

    def per_item(m):
        full = (ncg - half) * (4 * ((m + 3) // 4)) * 32
        tail = half * (8 * ((m + 7) // 8)) * 16
        return (full + tail) * rows

    return float(((items - 1) * per_item(mbig) + per_item(m_last)).sum())


def ncu_traffic(kernel: str, config: str | None = None):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch from the
    committed `ncu --set full` capture of this kernel on this workload
    (`kernel@config` first, then the kernel's generic entry)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None, None
    with open(p) as f:
        table = json.load(f)
    d = table.get(f"{kernel}@{config}") if config else None
    if d is None:
        d = table.get(kernel)
    return (d["dram_bytes_per_launch"], d["source"]) if d else (None, None)


def kernel_for(o, batch):
    """The query kernel psp_gpu_query_batch_device picks for a batch
    (engine_oracle.cuh launch_queries): query_cta below CTA_MAX_DENSITY
    queries per component pair, else query_grouped; PSP_QUERY_KERNEL
    overrides."""
    import paper_1503_07192_b200 as P
    forced = os.environ.get("PSP_QUERY_KERNEL")
    if forced in ("warp", "grouped", "cta"):
        return forced
    pairs = o.k * (o.k + 1) / 2
    return ("cta" if batch < P.CTA_MAX_DENSITY * pairs or batch <= P.CTA_MAX_COUNT
            else "grouped")


def launches_per_batch(o, batch):
    """Kernels one psp_gpu_query_batch_device call launches (all ours,
    cub's scan is compiled into libpsp_gpu.so): the grouped path runs
    group_prep, group_tasks, 2 x (cub ScanInit + Scan), group_emit,
    group_scatter, query_grouped, group_finish; query_cta / query_warp run
    alone (engine_oracle.cuh launch_grouped / launch_queries)."""
    import paper_1503_07192_b200 as P
    if kernel_for(o, batch) != "grouped":
        return 1
    # sparse grouping: cub radix sort (onesweep: histogram + 3 passes for the
    # <= 24-bit pair keys) and run-length encode (3) replace the bin pass
    sparse = (o.k * o.k >= P.SPARSE_GROUPING_MIN_BINS
              and batch * P.SPARSE_GROUPING_RATIO < o.k * o.k)
    return 16 if sparse else 10


def roofline_entry(o, batch, steps, tb, tops, per_launch_ms, peaks, peak_u32, world,
                   peak_insn="VIADDMNMX.U32", config=None, texec=None):
    """Dominant kernel of the query step. Dense batches (>= 2 queries per
    component pair) run query_grouped, which reuses each pair's boundary
    block from shared memory: it is bound by the min-plus ALU rate, so
    `achieved` is useful relaxations (B1*B2 + B2 per query, the reference's
    minplus_ops) per second per GPU against the in-run VIADDMNMX peak; the
    no-reuse HBM figure is reported beside it, never as a fraction > 1.
    Sparse batches run query_warp, which is HBM bound."""
    dense = kernel_for(o, batch) == "grouped"
    secs = per_launch_ms / 1e3
    ops_launch = tops / steps
    bytes_launch = tb / steps
    if dense:
        traffic, src = ncu_traffic("query_grouped", config)
        ach = ops_launch / secs
        return {"kernel": "query_grouped (K3, dense batch)", "bound": "alu",
                "achieved": round(ach / 1e12, 4), "peak": round(peak_u32 / 1e12, 4),
                "unit": "T relax/s", "frac": round(ach / peak_u32, 4),
                "traffic": traffic, "traffic_source": src,
                "peak_source": f"in-run min-plus probe ({peak_insn}), see profiles/r1_minplus_peak.json",
                "ops_per_query": round(ops_launch / batch, 1),
                # the kernel's own ALU rate: executed relaxations incl. the
                # lane layout's padding (grouped_executed_relaxations; within
                # 0.5% of ncu's VIADDMNMX count x 32 at cfg3)
                "executed_frac": round(texec / steps / secs / peak_u32, 4) if texec else None,
                "useful_share_of_executed": round(tops / texec, 4) if texec else None,
                "no_reuse_bytes_per_query": round(bytes_launch / batch, 1),
                "no_reuse_equiv_gbs": round(bytes_launch / secs / 1e9, 1),
                "hbm_peak_gbs": peaks["hbm_gbs"]}
    kname = "query_" + kernel_for(o, batch)
    traffic, src = ncu_traffic(kname, config)
    ach = bytes_launch / secs / 1e9
    return {"kernel": f"{kname} (K3, sparse batch)", "bound": "hbm", "achieved": round(ach, 1),
            "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": round(ach / peaks["hbm_gbs"], 4),
            "traffic": traffic, "traffic_source": src, "peak_source": peaks["source"],
            "bytes_per_query": round(bytes_launch / batch, 1)}


# ---------------------------------------------------------------- ours ----
def run_ours(args, rank, world, local):
    import torch
    import paper_1503_07192_b200 as P
    from paper_1503_07192_b200 import graphs

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        # the library's own NCCL communicator shards the boundary-graph FW
        obj = [P.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ctx = P.Context(local, rank, world, obj[0])
    else:
        ctx = P.Context(local)

    # process warm-up outside the timed build: one small oracle (64x64 grid,
    # k = 16, f32 and u32) loads the kernel modules lazily and primes the
    # allocator, as the warm-up steps do for the queries
    wg = P.generate_grid(64, 64, (1, 1025), 1)
    P.build_oracle(wg, 16, 1, 0, ctx=ctx)
    P.build_oracle(wg, 16, 1, 0, value_kind=P.VALUE_F32, ctx=ctx)
    t0 = time.time()
    g, cfg = graphs.make(args.config)
    gen_s = time.time() - t0
    threads = os.cpu_count() or 8

    def alloc_stats():
        out = np.zeros(4, np.uint64)
        P._lib.check(P._lib.lib().psp_gpu_alloc_stats(out))
        return out.astype(np.float64)

    alloc0 = alloc_stats()
    if world > 1:
        # one host partition (all cores, rank 0), broadcast, then the
        # collective device build with the boundary-graph FW row-sharded
        import torch.distributed as dist
        part = torch.empty(g.n, dtype=torch.int32, device=dev)
        part_s = 0.0
        if rank == 0:
            t0 = time.time()
            a = P.partition_graph(g, cfg["k"], 0, threads)
            part_s = time.time() - t0
            part.copy_(torch.from_numpy(a.view(np.int32)))
        dist.broadcast(part, src=0)
        o = P.build_partitioned(g, cfg["k"], part.cpu().numpy().view(np.uint32), ctx=ctx)
        o.stats["partition_ms"] = part_s * 1e3 + o.stats["partition_ms"]
    else:
        o = P.build_oracle(g, cfg["k"], threads, 0, ctx=ctx)
    st = o.stats
    alloc = alloc_stats() - alloc0  # host time inside cudaMalloc / cudaFree during the build

    stream = torch.cuda.Stream(device=dev)
    batch = args.batch or cfg["queries"]
    nsteps = args.warmup + args.steps
    # distinct pair slices per step and per rank (weak scaling)
    v1, v2 = P.random_pairs(g.n, batch * nsteps, 1000 + rank)
    d_v1 = torch.from_numpy(v1.view(np.int32)).to(dev)
    d_v2 = torch.from_numpy(v2.view(np.int32)).to(dev)
    d_out = torch.empty(batch, dtype=torch.float64, device=dev)

    def step(i):
        o.batch_query_device(d_v1[i * batch:].data_ptr(), d_v2[i * batch:].data_ptr(),
                             d_out.data_ptr(), batch, stream.cuda_stream)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    # the sampler runs from the warm-up through the timed region so that
    # even a sub-second region carries clock evidence
    with ClockSampler(local) as clk:
        for i in range(args.warmup):
            step(i)
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        for i in range(args.warmup, nsteps):
            step(i)
        ev1.record(stream)
        torch.cuda.synchronize()
    dev_ms = ev0.elapsed_time(ev1)
    barrier()
    # algorithmic bytes of the timed launches
    tb, tops = query_bytes_and_ops(o, v1[args.warmup * batch:], v2[args.warmup * batch:])
    texec = None
    if kernel_for(o, batch) == "grouped":
        # executed (padded) relaxations: exact for the first timed batch, the
        # others are draws of the same distribution (x steps)
        comp = o.assignment[o.permutation]
        bsize = np.diff(o.boundary_offset).astype(np.int64)
        i0 = args.warmup * batch
        texec = args.steps * grouped_executed_relaxations(o.k, bsize, comp[v1[i0:i0 + batch]],
                                                          comp[v2[i0:i0 + batch]])
        tops0 = query_bytes_and_ops(o, v1[i0:i0 + batch], v2[i0:i0 + batch])[1]
        texec *= (tops / args.steps) / tops0  # same useful work as the timed steps on average

    # ---- e2e through the public host API (pinned host buffers)
    h_v1 = torch.from_numpy(v1.view(np.int32)).pin_memory()
    h_v2 = torch.from_numpy(v2.view(np.int32)).pin_memory()
    h_out = torch.empty(batch, dtype=torch.float64).pin_memory()
    lib = P._lib.lib()

    # (1) synchronous host API, one batch per call (psp_gpu_query_batch)
    def e2e_sync_step(i):
        P._lib.check(lib.psp_gpu_query_batch(
            o.h, batch, h_v1[i * batch:].data_ptr(), h_v2[i * batch:].data_ptr(),
            h_out.data_ptr(), None))

    for i in range(args.warmup):
        e2e_sync_step(i)
    barrier()
    t_e = time.perf_counter()
    for i in range(args.warmup, nsteps):
        e2e_sync_step(i)
    e2e_sync_ms = (time.perf_counter() - t_e) * 1e3
    barrier()

    # (2) the pipelined host API (psp_gpu_query_pipe_*, 2 batches in
    # flight): every step still copies its pairs in and its distances out
    # inside the timed region; the copies of neighbouring steps overlap the
    # kernels. The region ends when the last batch's distances are on the host.
    depth = 2
    pipe = o.query_pipe(depth)
    h_outs = [torch.empty(batch, dtype=torch.float64).pin_memory() for _ in range(depth)]

    def e2e_step(i):
        pipe.submit(h_v1[i * batch:].data_ptr(), h_v2[i * batch:].data_ptr(),
                    h_outs[i % depth].data_ptr(), count=batch)

    for i in range(args.warmup):
        e2e_step(i)
    pipe.wait()
    barrier()
    t_e = time.perf_counter()
    for i in range(args.warmup, nsteps):
        e2e_step(i)
    pipe.wait()
    e2e_ms = (time.perf_counter() - t_e) * 1e3
    barrier()
    assert np.array_equal(h_outs[(nsteps - 1) % depth].numpy(), h_out.numpy()), "pipe/sync mismatch"
    pipe.close()

    # correctness spot check of the last batch against the e2e path
    ref_last = h_out.numpy().copy()
    step(nsteps - 1)
    torch.cuda.synchronize()
    assert np.array_equal(d_out.cpu().numpy(), ref_last), "device/e2e query mismatch"

    # max over ranks
    vals = torch.tensor([dev_ms, e2e_ms, st["k2_device_ms"], st["k1_device_ms"], e2e_sync_ms],
                        dtype=torch.float64, device=dev)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    dev_ms, e2e_ms, k2_ms, k1_ms, e2e_sync_ms = vals.tolist()

    if rank != 0:
        return None
    peaks = measured_peaks()
    total_q = batch * args.steps * world
    qps = total_q / (dev_ms / 1e3)
    e2e_qps = total_q / (e2e_ms / 1e3)
    per_launch_ms = dev_ms / args.steps
    achieved_gbs = (tb / args.steps) / (per_launch_ms / 1e3) / 1e9
    # the min-plus ALU peak of the arithmetic the tables use: VIADDMNMX.U32
    # (u32 fixed point) or FADD + FMNMX3 (f32)
    peak_u32, clock_mhz = ctx.minplus_peak(o.value_kind)
    peak_insn = "VIADDMNMX.U32" if o.value_kind == P.VALUE_U32 else "FADD+FMNMX3.F32"
    if o.value_kind != P.VALUE_U32:
        # the standalone probe's register allocation reaches a higher f32
        # rate than the in-library one; the larger figure is the denominator
        try:
            with open(os.path.join(ROOT, "profiles", "r1_minplus_peak.json")) as f:
                sa = json.load(f)["variants"]["f32_fadd_fmnmx3"]["relax_per_s"]
            if sa > peak_u32:
                peak_u32 = sa
                peak_insn += ", standalone tools/minplus_probe figure (higher than in-run)"
        except (OSError, KeyError, ValueError):
            pass
    k2_rate = st["k2_relaxations"] / (k2_ms / 1e3) if k2_ms else 0.0  # max over ranks
    bg_gb = o.b * (o.b + 128) * 2 / 1e9
    line = {
        "metric": METRIC,
        "value": round(qps, 1),
        "unit": "queries/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(dev_ms / args.steps, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u32" if o.value_kind == P.VALUE_U32 else "f32",
        "data": f"synthetic (seeded {FAMILY[cfg['family']]} graph + mt19937_64 pairs)",
        "config": workload_config(args.config, cfg, g.n, batch),
        "parallelism": (f"boundary-graph FW row-sharded over {world} GPUs (NCCL panel "
                        f"exchange), queries sharded by rank, tables replicated"
                        if world > 1 else "1 GPU"),
        "tables": {"b": o.b, "m": g.m, "boundary_table_gb": round(bg_gb, 2),
                   "value_kind": "u32" if o.value_kind == P.VALUE_U32 else "f32"},
        "e2e": {"value": round(e2e_qps, 1), "unit": "queries/s",
                "h2d_bytes_per_step": 8 * batch, "d2h_bytes_per_step": 8 * batch,
                "api": f"psp_gpu_query_pipe_submit/wait ({depth} batches in flight, pinned host "
                       "pairs in, f64 distances out, copies overlapped with the kernels)",
                "sync_api_value": round(total_q / (e2e_sync_ms / 1e3), 1),
                "sync_api": "psp_gpu_query_batch (one blocking call per step)"},
        "gpu_launches": args.steps * launches_per_batch(o, batch),
        "roofline": roofline_entry(o, batch, args.steps, tb, tops, per_launch_ms, peaks,
                                   peak_u32, world, peak_insn, args.config, texec),
        "preprocessing": {
            "graph_gen_s": round(gen_s, 2),
            "partition_s": round(st["partition_ms"] / 1e3, 3),
            "component_apsp_s": round(st["component_apsp_ms"] / 1e3, 3),
            "boundary_s": round(st["boundary_ms"] / 1e3, 3),
            "preprocessing_s": round((st["partition_ms"] + st["component_apsp_ms"]
                                      + st["boundary_ms"]) / 1e3, 3),
            "host_subphases_s": {"split": round(st["split_ms"] / 1e3, 3),
                                 "k1_order": round(st["k1_order_ms"] / 1e3, 3),
                                 "k2_order_layout": round(st["bg_order_ms"] / 1e3, 3)},
            "boundary_minus_k2_device_s": round((st["boundary_ms"] - st["k2_device_ms"]) / 1e3, 3),
            # driver time inside the build's cudaMalloc / cudaFree calls (single
            # calls have stalled for 0.1-1 s on these boxes: the wall-clock noise)
            "driver_alloc": {"malloc_s": round(alloc[0] / 1e9, 3), "malloc_calls": int(alloc[1]),
                             "free_s": round(alloc[2] / 1e9, 3), "free_calls": int(alloc[3])},
            "k2_positions": st["k2_positions"],
            "k1_device_s": round(k1_ms / 1e3, 4), "k2_device_s": round(k2_ms / 1e3, 4),
            "k2_relax_per_s": k2_rate, "k2_alu_frac_per_gpu": round(k2_rate / (peak_u32 * world), 4),
            "minplus_peak_relax_per_s": peak_u32, "peak_source": "measured in-run "
            f"(minplus_peak_kernel, {peak_insn})", "host_threads": threads,
            "warmup_build": "one 64x64-grid oracle (u32 and f32) built before the timed build",
            "b": o.b, "bg_edges": st["bg_edges"], "stored_entries": st["stored_entries"]},
        "clocks": clk.summary(),
    }
    if args.cpu_baseline and world == 1:
        line["cpu_baseline"] = cpu_baseline(o, g, cfg, args)
    return line


# ----------------------------------------------------------- reference ----
def ref_workload(name: str):
    """The configuration's graph, drawn WITHOUT the product package:
    workloads.py (numpy/scipy) or, for the grid family, the reference's own
    generate_grid."""
    import oracle
    import workloads
    R = oracle.RefLib()

    def grid(rows, cols, weights, seed):
        rg = R.generate("grid", rows, cols, weights, seed)
        eu, ev, ew = rg.edges()
        return rg.n, eu, ev, ew

    (n, eu, ev, ew), cfg = workloads.make_arrays(name, grid=grid)
    return R, R.graph(n, eu, ev, ew), cfg


def sampled_pairs(ro, comps, count: int, seed: int, both: bool = False):
    """Uniform random pairs conditioned on the source lying in one of the
    sampled components (the only rows a sampled reference oracle holds):
    v1 uniform over those components' vertices, v2 uniform over all (or,
    `both`, over the same components: when not even every component table
    fits host RAM, the reference's col2 rows must come from sampled ones)."""
    assign_orig = ro.assignment[ro.permutation]  # original id -> component
    members = np.flatnonzero(np.isin(assign_orig, comps)).astype(np.uint32)
    rng = np.random.default_rng(seed)
    v1 = members[rng.integers(0, len(members), count)]
    v2 = (members[rng.integers(0, len(members), count)] if both
          else rng.integers(0, ro.n, count).astype(np.uint32))
    return v1, v2


def reference_build(rg, cfg, cores):
    """Reference preprocessing: build_oracle in full where its tables fit
    the host, else Phases 1-2 in full + Phase 3 on REF_COMPONENTS seeded
    components (ref_sampled_oracle). Returns (oracle, sampled components or
    None, preprocessing dict)."""
    if rg.n <= REF_FULL_MAX_N:
        t0 = time.time()
        ro = rg.build_oracle(cfg["k"], cores, 0)
        wall = time.time() - t0
        st = ro.stats
        return ro, None, {
            "mode": "full build_oracle", "workers": cores, "build_s": round(wall, 2),
            "partition_s": round(st["partition_ms"] / 1e3, 3),
            "component_apsp_s": round(st["component_apsp_ms"] / 1e3, 3),
            "boundary_s": round(st["boundary_ms"] / 1e3, 3), "b": ro.b}
    ro, comps, t = rg.sampled_oracle(cfg["k"], cores, REF_COMPONENTS, 0, 1)
    # boundary_apsp does |B(C)| Dijkstra rows per component on `cores`
    # threads; the sampled rows ran on the same threads, so wall time
    # scales with the row count
    boundary_s = (t["bg_build_ms"] + t["sampled_rows_ms"] * t["b"] / max(t["rows"], 1)) / 1e3
    return ro, comps, {
        "mode": (f"Phases 1-2 in full; Phase 3: build_boundary_graph in full + dijkstra_sssp "
                 f"rows of {len(comps)} seeded components ({t['rows']} of b={t['b']} rows), "
                 f"extrapolated x b/rows"),
        "workers": cores,
        "partition_s": round(t["partition_ms"] / 1e3, 3),
        "component_apsp_s": round(t["component_apsp_ms"] / 1e3, 3),
        "boundary_s": round(boundary_s, 2), "boundary_s_kind": "extrapolated",
        "boundary_graph_build_s": round(t["bg_build_ms"] / 1e3, 3),
        "sampled_rows": t["rows"], "sampled_rows_s": round(t["sampled_rows_ms"] / 1e3, 3),
        "build_s": round((t["partition_ms"] + t["component_apsp_ms"]) / 1e3 + boundary_s, 2),
        "build_s_kind": "measured phases 1-2 + extrapolated phase 3", "b": t["b"],
        "bg_edges": t["bg_edges"]}


def run_reference(args, rank, world):
    """The reference's own CPU implementation of the path (oracle/_ref,
    unmodified sources) on this box's host cores, on our arm's config and
    metric; each step is a bounded sample of the workload (args.ref_sample
    pairs through psp::batch_query with all cores)."""
    if rank != 0:
        return None
    cores = os.cpu_count() or 1
    # the reference's Phase 2 keeps every component table in f64 (~n^2/k x 8
    # bytes) and runs apsp_dense on each: beyond host RAM (road4m: ~260 GB,
    # and hours of CPU) no bounded sample of its own code path exists here
    import workloads
    cfg0 = workloads.CONFIGS[args.config]
    n0 = cfg0.get("n") or cfg0.get("rows", 0) * cfg0.get("cols", 0)
    # (and ~(n/k)^3 x k relaxations at ~4e9 per second per thread)
    mem_gb = float(n0) ** 2 / cfg0["k"] * 8 / 1e9 if n0 else 0.0
    cpu_s = float(n0) ** 3 / cfg0["k"] ** 2 / (4e9 * cores) if n0 else 0.0
    if mem_gb * 1e9 > 0.3 * host_mem_bytes() or cpu_s > 600:
        return {"impl": "reference", "unavailable": (
            f"{args.config}: the reference's Phase 2 holds all component tables in f64 "
            f"(~{mem_gb:.0f} GB) and takes ~{cpu_s / 60:.0f} min of apsp_dense on {cores} "
            f"threads; the reference arm runs configs up to delaunay1m_k1024")}
    t0 = time.time()
    R, rg, cfg = ref_workload(args.config)
    gen_s = time.time() - t0
    ro, comps, prep = reference_build(rg, cfg, cores)
    sample = args.ref_sample
    nsteps = args.warmup + args.steps
    if comps is None:
        v1, v2 = R.random_pairs(rg.n, sample * nsteps, 1000)
        pairs_desc = "uniform random pairs (ref::random_pairs)"
    else:
        v1, v2 = sampled_pairs(ro, comps, sample * nsteps, 1000)
        pairs_desc = (f"uniform random pairs with the source in the {len(comps)} sampled "
                      f"components (the reference's f64 boundary tables do not fit host RAM)")
    for i in range(args.warmup):
        ro.batch_query(v1[i * sample:(i + 1) * sample], v2[i * sample:(i + 1) * sample], cores)
    t0 = time.perf_counter()
    for i in range(args.warmup, nsteps):
        ro.batch_query(v1[i * sample:(i + 1) * sample], v2[i * sample:(i + 1) * sample], cores)
    dt = time.perf_counter() - t0
    qps = sample * args.steps / dt
    batch = args.batch or cfg["queries"]
    return {
        "impl": "reference", "metric": METRIC, "value": round(qps, 1), "unit": "queries/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(dt * 1e3 / args.steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (seeded {FAMILY[cfg['family']]} graph + mt19937_64 pairs)",
        "config": workload_config(args.config, cfg, rg.n, batch),
        "cpu_baseline": {"value": round(qps, 1), "unit": "queries/s", "cores": cores,
                         "kind": "reference",
                         "sample": f"{sample} pairs per step ({pairs_desc}), psp::batch_query "
                                   f"with {cores} threads, unmodified reference build"},
        "e2e": {"value": round(qps, 1), "unit": "queries/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "preprocessing": dict(prep, graph_gen_s=round(gen_s, 2)),
    }


def host_mem_bytes() -> float:
    """MemAvailable of this host (bytes)."""
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable:"):
                    return float(line.split()[1]) * 1024
    except OSError:
        pass
    return float(os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES"))


def cpu_baseline(o, g, cfg, args, sample=100_000, steps=3):
    """The reference's own query code (oracle/_ref, unmodified psp::batch_query)
    on this box's host cores, over a bounded sample of the same workload. The
    reference's preprocessing is timed by `--impl reference`; here its
    psp::Oracle is assembled from the GPU build's exported f64 tables (bit-
    identical to the reference's, tests/test_large_configs.py), with boundary
    rows for REF_COMPONENTS seeded components where all of them would not
    fit host RAM; pairs then start in those components."""
    import oracle
    R = oracle.RefLib()
    cores = os.cpu_count() or 1
    t0 = time.time()
    k = o.k
    full = g.n <= REF_FULL_MAX_N
    rng = np.random.default_rng(1)
    comps = np.arange(k) if full else np.sort(rng.choice(k, REF_COMPONENTS, replace=False))
    cs = set(comps.tolist())
    # every component table in f64 (the reference's col2 rows come from
    # them) unless that would not fit host RAM comfortably (road4m: 275 GB);
    # then only the sampled components', and both query ends in them
    csize = np.diff(o.component_offset).astype(np.float64)
    both = not full and float((csize ** 2).sum()) * 8 > 0.3 * host_mem_bytes()
    ct = [o.component_table(c) if (c in cs or not both) else None for c in range(k)]
    bt = [o.boundary_rows(c) if c in cs else None for c in range(k)]
    ro = oracle.assemble_oracle(R, g.n, k, o.permutation, o.assignment, o.boundary_flags,
                                o.component_offset, o.boundary_offset, o.boundary_vertex, ct, bt)
    del ct, bt
    export_s = time.time() - t0
    if full:
        v1, v2 = R.random_pairs(g.n, sample * (steps + 1), 77)
    else:
        v1, v2 = sampled_pairs(ro, comps, sample * (steps + 1), 77, both)
    ro.batch_query(v1[:sample], v2[:sample], cores)  # warm-up
    t0 = time.perf_counter()
    d = ro.batch_query(v1[sample:], v2[sample:], cores)
    qs = sample * steps / (time.perf_counter() - t0)
    # the GPU answers the same pairs: bit for bit in u32, within the f32
    # tolerance (relative 1e-5, BASELINE north_star) otherwise
    dg = o.batch_query(v1[sample:], v2[sample:])
    import paper_1503_07192_b200 as P
    if o.value_kind == P.VALUE_U32:
        assert np.array_equal(dg, d), "GPU != reference"
    else:
        assert np.allclose(dg, d, rtol=1e-5, atol=0), "GPU != reference within 1e-5"
    return {"value": round(qs, 1), "unit": "queries/s", "cores": cores, "kind": "reference",
            "sample": (f"{sample * steps} random pairs"
                       + ("" if full else f" with the {'source and target' if both else 'source'} "
                                          f"in {REF_COMPONENTS} seeded components")
                       + f", psp::batch_query with {cores} threads on a psp::Oracle assembled "
                         f"from the GPU build's f64 exports ({export_s:.1f} s); answers checked "
                         f"equal to the GPU's" + ("" if o.value_kind == P.VALUE_U32 else
                                                  " within relative 1e-5 (f32 path)")
                       + ". Reference preprocessing: see --impl reference")}


def workload_config(name, cfg, n, batch):
    """`config` of both arms (identical by construction)."""
    return {"workload": f"{name}: {FAMILY[cfg['family']]} n={n} k={cfg['k']}, {batch} random "
                        f"pairs per step per GPU", "batch_per_gpu": batch,
            "l2_policy": "inputs >> L2 (boundary-graph table >> 126 MB), fresh pairs each step"
                         if n > 100_000 else "small config: tables may fit in L2"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default=CONFIG)
    ap.add_argument("--batch", type=int, default=0,
                    help="pairs per step per GPU (default: the config's query count)")
    ap.add_argument("--ref-sample", type=int, default=100_000)
    ap.add_argument("--cpu-baseline", dest="cpu_baseline", action="store_true", default=True)
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    rank, world, local = dist_env()
    # stdout carries exactly the one JSON line: anything the libraries print
    # there (NCCL's version banner on communicator init, ...) goes to stderr
    sys.stdout.flush()
    json_fd = os.dup(1)
    os.dup2(2, 1)
    if args.impl == "reference":
        line = run_reference(args, rank, world)
    else:
        line = run_ours(args, rank, world, local)
    sys.stdout.flush()
    if line is not None:
        os.write(json_fd, (json.dumps(line) + "\n").encode())


if __name__ == "__main__":
    main()
