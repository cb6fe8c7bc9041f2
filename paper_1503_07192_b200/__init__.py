"""B200-native preprocessing + query engine for the partitioned planar
shortest-path oracle (Chapuis & Djidjev, arXiv 1503.07192).

Host-side mirror of the reference library's hot-path interface
(/root/reference/proj/include/psp): ``build_oracle`` (oracle.hpp:85-86),
``query`` / ``batch_query`` (query.hpp:36-46), ``apsp_dense``
(shortest_paths.hpp:43), ``boundary_apsp`` (oracle.hpp:94-96),
``partition_graph`` (partition.hpp:42) and the grid generators
(generators.hpp:24-30). Everything computes through the C-ABI library
``libpsp_gpu.so`` (include/psp_gpu.h) on a B200; errors follow the
reference: bad arguments raise ``ValueError`` (std::invalid_argument), graph
invariant violations raise :class:`GraphInvariantError`.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os

import numpy as np

from . import _lib
from ._lib import (VALUE_AUTO, VALUE_F32, VALUE_U32, BuildStats, ChecksumError,
                   FormatVersionError, GraphInvariantError, OracleIoError, ParseError, PspError,
                   PspValueError)

from . import cluster  # noqa: E402  (placement + routed queries, cluster.hpp)
from .cluster import (PAIRS_PER_GPU, ROUND_ROBIN, Placement, RoutedOracle,  # noqa: E402
                      TransferLedger, TransferRecord, place_components, routed_query,
                      simulate_build_schedule)

__all__ = ["load_graph", "read_graph", "save_graph", "write_graph", "format_weight",
           "ParseError", "EDGE_LIST", "DIMACS", "cluster", "Placement", "RoutedOracle", "TransferLedger", "TransferRecord",
           "place_components", "routed_query", "simulate_build_schedule", "ROUND_ROBIN",
           "PAIRS_PER_GPU", "Graph", "Context", "nccl_unique_id", "import_oracle", "GpuOracle", "build_oracle", "build_partitioned", "apsp_dense",
           "boundary_apsp", "partition_graph", "generate_grid", "generate_triangulated_grid",
           "random_pairs", "VALUE_AUTO", "VALUE_U32", "VALUE_F32", "PspError", "PspValueError",
           "GraphInvariantError", "OracleIoError", "FormatVersionError", "ChecksumError",
           "load_oracle", "UNREACHABLE", "STORAGE_REPLICATED", "STORAGE_ROW_SHARDED"]

UNREACHABLE = float("inf")  # kUnreachable (include/psp/graph.hpp:14)
# boundary-graph table storage of multi-GPU builds (psp_boundary_storage)
STORAGE_REPLICATED = 0
STORAGE_ROW_SHARDED = 1
# batch density (queries per component pair c1 <= c2) rules of the query
# launcher (must match engine_oracle.cuh): below CTA_MAX_DENSITY a batch runs
# query_cta (one CTA per query, no sort), else the pair-grouped kernel
GROUP_MIN_DENSITY = 0.0
CTA_MAX_DENSITY = 0.0
CTA_MAX_COUNT = 16384        # batches up to this size: query_cta (one launch)
SPARSE_GROUPING_RATIO = 4    # grouped batches with count * 4 < k^2 ...
SPARSE_GROUPING_MIN_BINS = 1 << 24  # ... and k^2 >= 2^24: radix-sort grouping


@dataclasses.dataclass
class Graph:
    """Undirected weighted edge list, each edge once (psp::Graph(n, edges))."""

    n: int
    eu: np.ndarray
    ev: np.ndarray
    ew: np.ndarray

    def __post_init__(self):
        self.eu = np.ascontiguousarray(self.eu, np.uint32)
        self.ev = np.ascontiguousarray(self.ev, np.uint32)
        self.ew = np.ascontiguousarray(self.ew, np.float64)

    @property
    def m(self) -> int:
        return len(self.eu)


class Context:
    """One GPU (one process per GPU). Owns the CUDA stream used by builds."""

    def __init__(self, device: int = 0, rank: int = 0, world: int = 1, nccl_id: bytes | None = None):
        h = C.c_void_p()
        buf = C.create_string_buffer(nccl_id, 128) if nccl_id else None
        _lib.check(_lib.lib().psp_gpu_ctx_create(device, rank, world, buf, C.byref(h)))
        self.h = h
        self.device, self.rank, self.world = device, rank, world

    def close(self):
        if getattr(self, "h", None):
            _lib.lib().psp_gpu_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self) -> int:
        return _lib.lib().psp_gpu_ctx_stream(self.h) or 0

    def set_boundary_storage(self, storage: int) -> None:
        """STORAGE_REPLICATED (default) or STORAGE_ROW_SHARDED for later
        multi-GPU builds (include/psp_gpu.h psp_gpu_ctx_set_boundary_storage):
        row-sharded oracles keep ~1/world of the boundary-graph table per GPU
        and answer through RoutedOracle only."""
        _lib.check(_lib.lib().psp_gpu_ctx_set_boundary_storage(self.h, int(storage)))

    def minplus_peak(self, value_kind: int = VALUE_U32):
        r, mhz = C.c_double(), C.c_double()
        _lib.check(_lib.lib().psp_gpu_minplus_peak(self.h, value_kind, C.byref(r), C.byref(mhz)))
        return r.value, mhz.value


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id for a multi-GPU Context (create on rank 0 and
    broadcast, e.g. with torch.distributed.broadcast_object_list)."""
    buf = C.create_string_buffer(128)
    _lib.check(_lib.lib().psp_gpu_nccl_unique_id(buf))
    return buf.raw


_default_ctx: Context | None = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


class GpuOracle:
    """Device-resident oracle (psp::Oracle, include/psp/oracle.hpp:47-78)."""

    def __init__(self, ctx: Context, h, stats: BuildStats):
        self.ctx, self.h = ctx, h
        self.stats = stats.as_dict()
        info = _lib.OracleInfo()
        _lib.check(_lib.lib().psp_gpu_oracle_info(h, C.byref(info)))
        self.n, self.k, self.b = int(info.n), int(info.k), int(info.b)
        self.value_kind = int(info.value_kind)
        self.fixed_point_shift = int(info.fixed_point_shift)
        self.tile = int(info.tile)
        n, k = self.n, self.k
        self.permutation = np.empty(n, np.uint32)
        self.inverse_permutation = np.empty(n, np.uint32)
        self.assignment = np.empty(n, np.uint32)       # reordered id space
        self.boundary_flags = np.empty(n, np.uint8)    # reordered id space
        self.component_offset = np.empty(k + 1, np.uint64)
        self.boundary_offset = np.empty(k + 1, np.uint64)
        self.boundary_vertex = np.empty(max(self.b, 1), np.uint32)
        p = lambda a: a.ctypes.data_as(C.c_void_p)
        _lib.check(_lib.lib().psp_gpu_oracle_ids(
            h, p(self.permutation), p(self.inverse_permutation), p(self.assignment),
            p(self.boundary_flags), p(self.component_offset), p(self.boundary_offset),
            p(self.boundary_vertex)))
        self.boundary_vertex = self.boundary_vertex[: self.b]

    def close(self):
        if getattr(self, "h", None):
            _lib.lib().psp_gpu_oracle_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- table access (Oracle::component_tables / boundary_tables) --------
    def component_size(self, c: int) -> int:
        return int(self.component_offset[c + 1] - self.component_offset[c])

    def boundary_size(self, c: int) -> int:
        return int(self.boundary_offset[c + 1] - self.boundary_offset[c])

    def stored_entries(self) -> int:
        s = np.diff(self.component_offset).astype(np.int64)
        bsz = np.diff(self.boundary_offset).astype(np.int64)
        return int((s * s).sum() + bsz.sum() * self.b)

    def component_table(self, c: int) -> np.ndarray:
        s = self.component_size(c)
        out = np.empty(max(s * s, 1), np.float64)
        _lib.check(_lib.lib().psp_gpu_export_component(self.h, c, out))
        return out[: s * s].reshape(s, s)

    def boundary_rows(self, c: int) -> np.ndarray:
        r = self.boundary_size(c)
        out = np.empty(max(r * self.b, 1), np.float64)
        _lib.check(_lib.lib().psp_gpu_export_boundary_rows(self.h, c, out))
        return out[: r * self.b].reshape(r, self.b)

    # -- queries (query.hpp:36-46) ----------------------------------------
    def batch_query(self, v1, v2, with_ops: bool = False):
        """Distances for original-id pairs, host arrays in/out (f64, +inf)."""
        v1 = np.ascontiguousarray(v1, np.uint32)
        v2 = np.ascontiguousarray(v2, np.uint32)
        if v1.shape != v2.shape:
            raise ValueError("batch_query: v1 and v2 differ in length")
        dist = np.empty(len(v1), np.float64)
        ops = np.empty(len(v1), np.uint64) if with_ops else None
        p = lambda a: a.ctypes.data_as(C.c_void_p) if a is not None else None
        _lib.check(_lib.lib().psp_gpu_query_batch(self.h, len(v1), p(v1), p(v2), p(dist), p(ops)))
        return (dist, ops) if with_ops else dist

    def query(self, v1: int, v2: int):
        d, ops = self.batch_query([v1], [v2], with_ops=True)
        return float(d[0]), int(ops[0])

    def save(self, path: str) -> None:
        """psp::save_oracle (include/psp/oracle_io.hpp:31): PSP1 file written
        from the device tables, byte-identical to the reference's image."""
        _lib.check(_lib.lib().psp_gpu_oracle_save(self.h, os.fsencode(path)))

    def query_pipe(self, depth: int = 2) -> "QueryPipe":
        """Pipelined host batches (psp_gpu_query_pipe_*): copies of
        neighbouring batches overlap the kernels of the current one."""
        return QueryPipe(self, depth)

    def batch_query_device(self, v1_ptr: int, v2_ptr: int, dist_ptr: int, count: int,
                           stream: int | None = None) -> None:
        """Device-resident queries: raw device pointers, enqueued on `stream`."""
        _lib.check(_lib.lib().psp_gpu_query_batch_device(self.h, count, v1_ptr, v2_ptr, dist_ptr,
                                                         stream))


class QueryPipe:
    """Up to `depth` host batches in flight on one oracle. submit() returns at
    once; the arrays passed to it are kept alive until wait(), which drains
    the pipe and raises ValueError if a batch held an id >= n (that batch's
    distances are then unspecified). Arrays may be numpy (copied to
    contiguous u32 / written in place as f64) or raw host pointers."""

    def __init__(self, oracle: "GpuOracle", depth: int = 2):
        self.oracle = oracle
        self.h = C.c_void_p()
        _lib.check(_lib.lib().psp_gpu_query_pipe_create(oracle.h, depth, C.byref(self.h)))
        self._live = []

    def submit(self, v1, v2, dist, count: int | None = None) -> None:
        if isinstance(v1, int):  # raw pointers
            _lib.check(_lib.lib().psp_gpu_query_pipe_submit(self.h, count, v1, v2, dist))
            return
        v1 = np.ascontiguousarray(v1, np.uint32)
        v2 = np.ascontiguousarray(v2, np.uint32)
        if v1.shape != v2.shape or dist.shape != v1.shape or dist.dtype != np.float64:
            raise ValueError("QueryPipe.submit: v1, v2, dist must have equal length (dist f64)")
        if not dist.flags.c_contiguous:
            raise ValueError("QueryPipe.submit: dist must be contiguous")
        self._live.append((v1, v2, dist))
        p = lambda a: a.ctypes.data_as(C.c_void_p)
        _lib.check(_lib.lib().psp_gpu_query_pipe_submit(self.h, len(v1), p(v1), p(v2), p(dist)))

    def wait(self) -> None:
        try:
            _lib.check(_lib.lib().psp_gpu_query_pipe_wait(self.h))
        finally:
            self._live.clear()

    def close(self) -> None:
        if self.h:
            _lib.lib().psp_gpu_query_pipe_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def build_oracle(g: Graph, k: int, workers: int = 1, seed: int = 0,
                 value_kind: int = VALUE_AUTO, ctx: Context | None = None) -> GpuOracle:
    """psp::build_oracle (include/psp/oracle.hpp:85-86) on the GPU."""
    ctx = ctx or default_context()
    h = C.c_void_p()
    st = BuildStats()
    _lib.check(_lib.lib().psp_gpu_build_oracle(ctx.h, g.n, g.m, g.eu, g.ev, g.ew, k, workers,
                                               seed, value_kind, C.byref(h), C.byref(st)))
    return GpuOracle(ctx, h, st)


def build_partitioned(g: Graph, k: int, assignment, value_kind: int = VALUE_AUTO,
                      ctx: Context | None = None) -> GpuOracle:
    """build with a caller-supplied assignment in original ids (make_partition)."""
    ctx = ctx or default_context()
    a = np.ascontiguousarray(assignment, np.uint32)
    if len(a) != g.n:
        raise ValueError("assignment must cover all vertices")
    h = C.c_void_p()
    st = BuildStats()
    _lib.check(_lib.lib().psp_gpu_build_partitioned(ctx.h, g.n, g.m, g.eu, g.ev, g.ew, k, a,
                                                    value_kind, C.byref(h), C.byref(st)))
    return GpuOracle(ctx, h, st)


def import_oracle(n: int, k: int, permutation, assignment_reordered, component_offset,
                  boundary_offset, component_tables, boundary_tables,
                  value_kind: int = VALUE_AUTO, ctx: Context | None = None) -> GpuOracle:
    """Device oracle from host tables (e.g. a psp::Oracle read by load_oracle,
    include/psp/oracle_io.hpp:22-34): psp_gpu_oracle_import."""
    ctx = ctx or default_context()
    perm = np.ascontiguousarray(permutation, np.uint32)
    asg = np.ascontiguousarray(assignment_reordered, np.uint32)
    co = np.ascontiguousarray(component_offset, np.uint64)
    bo = np.ascontiguousarray(boundary_offset, np.uint64)
    cts = [np.ascontiguousarray(t, np.float64) for t in component_tables]
    bts = [np.ascontiguousarray(t, np.float64) for t in boundary_tables]
    if len(cts) != k or len(bts) != k:
        raise ValueError("one component table and one boundary table per component")
    cp = (C.c_void_p * k)(*[t.ctypes.data for t in cts])
    bp = (C.c_void_p * k)(*[t.ctypes.data for t in bts])
    h = C.c_void_p()
    _lib.check(_lib.lib().psp_gpu_oracle_import(ctx.h, n, k, perm, asg, co, bo, cp, bp,
                                                value_kind, C.byref(h)))
    return GpuOracle(ctx, h, BuildStats())


def load_oracle(path: str, value_kind: int = VALUE_AUTO, ctx: Context | None = None) -> GpuOracle:
    """psp::load_oracle (include/psp/oracle_io.hpp:32) into device memory."""
    ctx = ctx or default_context()
    h = C.c_void_p()
    _lib.check(_lib.lib().psp_gpu_oracle_load(ctx.h, os.fsencode(path), value_kind, C.byref(h)))
    return GpuOracle(ctx, h, BuildStats())


def apsp_dense(g: Graph, block_size: int = 64, value_kind: int = VALUE_AUTO,
               ctx: Context | None = None) -> np.ndarray:
    """psp::apsp_dense (include/psp/shortest_paths.hpp:43) on the GPU."""
    ctx = ctx or default_context()
    out = np.empty(max(g.n * g.n, 1), np.float64)
    _lib.check(_lib.lib().psp_gpu_apsp_dense(ctx.h, g.n, g.m, g.eu, g.ev, g.ew, block_size,
                                             value_kind, out))
    return out[: g.n * g.n].reshape(g.n, g.n)


def boundary_apsp(bg: Graph, value_kind: int = VALUE_AUTO, ctx: Context | None = None):
    """psp::boundary_apsp (include/psp/oracle.hpp:94-96): the b x b table,
    rows in boundary-id order (the reference's per-component matrices
    concatenated)."""
    ctx = ctx or default_context()
    out = np.empty(max(bg.n * bg.n, 1), np.float64)
    _lib.check(_lib.lib().psp_gpu_boundary_apsp(ctx.h, bg.n, bg.m, bg.eu, bg.ev, bg.ew,
                                                value_kind, out))
    return out[: bg.n * bg.n].reshape(bg.n, bg.n)


def partition_graph(g: Graph, k: int, seed: int = 0, threads: int = 8) -> np.ndarray:
    """psp::partition_graph (include/psp/partition.hpp:42): assignment only."""
    a = np.empty(g.n, np.uint32)
    _lib.check(_lib.lib().psp_partition_graph(g.n, g.m, g.eu, g.ev, g.ew, k, seed, threads, a))
    return a


def _grid(kind: int, rows: int, cols: int, weights, seed: int) -> Graph:
    unit = 1 if weights is None else 0
    lo, hi = (1.0, 1.0) if weights is None else (float(weights[0]), float(weights[1]))
    m = C.c_uint64()
    _lib.check(_lib.lib().psp_generate_grid(kind, rows, cols, unit, lo, hi, seed, C.byref(m),
                                            None, None, None))
    eu = np.empty(m.value, np.uint32)
    ev = np.empty(m.value, np.uint32)
    ew = np.empty(m.value, np.float64)
    p = lambda a: a.ctypes.data_as(C.c_void_p)
    _lib.check(_lib.lib().psp_generate_grid(kind, rows, cols, unit, lo, hi, seed, C.byref(m),
                                            p(eu), p(ev), p(ew)))
    return Graph(rows * cols, eu, ev, ew)


def generate_grid(rows: int, cols: int, weights=None, seed: int = 0) -> Graph:
    """psp::generate_grid; weights None = unit, (lo, hi) = uniform lattice."""
    return _grid(0, rows, cols, weights, seed)


def generate_triangulated_grid(rows: int, cols: int, weights=None, seed: int = 0) -> Graph:
    """psp::generate_triangulated_grid."""
    return _grid(1, rows, cols, weights, seed)


# ------------------------------------------------------- graph ingestion --
# psp::FileFormat (include/psp/graph_io.hpp:10-13)
EDGE_LIST, DIMACS = "edge_list", "dimacs"
_FORMATS = {EDGE_LIST: _lib.FORMAT_EDGE_LIST, DIMACS: _lib.FORMAT_DIMACS}


def _format(fmt: str) -> int:
    if fmt not in _FORMATS:
        raise ValueError(f"unknown graph format {fmt!r} (edge_list | dimacs)")
    return _FORMATS[fmt]


def _take_graph(h) -> Graph:
    L = _lib.lib()
    n, m = C.c_uint64(), C.c_uint64()
    try:
        _lib.check(L.psp_graph_size(h, C.byref(n), C.byref(m)))
        eu = np.empty(max(m.value, 1), np.uint32)
        ev = np.empty(max(m.value, 1), np.uint32)
        ew = np.empty(max(m.value, 1), np.float64)
        p = lambda a: a.ctypes.data_as(C.c_void_p)
        _lib.check(L.psp_graph_edges(h, p(eu), p(ev), p(ew)))
    finally:
        L.psp_graph_free(h)
    k = m.value
    return Graph(int(n.value), eu[:k], ev[:k], ew[:k])


def load_graph(path: str, fmt: str = EDGE_LIST, ctx: Context | None = None) -> Graph:
    """psp::load_graph (graph_io.hpp:18): the file is parsed on the GPU.
    Raises ParseError / GraphInvariantError / OracleIoError as the reference
    throws ParseError / GraphInvariantError / IoError."""
    ctx = ctx or default_context()
    h = C.c_void_p()
    _lib.check(_lib.lib().psp_gpu_load_graph(ctx.h, os.fsencode(path), _format(fmt), C.byref(h)))
    return _take_graph(h)


def read_graph(text, fmt: str = EDGE_LIST, name: str = "<stream>",
               ctx: Context | None = None) -> Graph:
    """psp::read_graph (graph_io.hpp:19) over in-memory text (str or bytes)."""
    ctx = ctx or default_context()
    data = text.encode() if isinstance(text, str) else bytes(text)
    h = C.c_void_p()
    _lib.check(_lib.lib().psp_gpu_read_graph(ctx.h, data, len(data), _format(fmt),
                                             name.encode(), C.byref(h)))
    return _take_graph(h)


def _edges(g: Graph):
    eu = np.ascontiguousarray(g.eu, np.uint32)
    ev = np.ascontiguousarray(g.ev, np.uint32)
    ew = np.ascontiguousarray(g.ew, np.float64)
    return eu, ev, ew, (lambda a: a.ctypes.data_as(C.c_void_p))


def write_graph(g: Graph, fmt: str = EDGE_LIST) -> str:
    """psp::write_graph (graph_io.hpp:22): the graph's sorted edge list as
    text, byte-identical to the reference's."""
    eu, ev, ew, p = _edges(g)
    L = _lib.lib()
    n = C.c_uint64()
    _lib.check(L.psp_write_graph(g.n, len(eu), p(eu), p(ev), p(ew), _format(fmt), None, 0,
                                 C.byref(n)))
    buf = C.create_string_buffer(max(n.value, 1))
    _lib.check(L.psp_write_graph(g.n, len(eu), p(eu), p(ev), p(ew), _format(fmt), buf, n.value,
                                 C.byref(n)))
    return buf.raw[: n.value].decode()


def save_graph(g: Graph, path: str, fmt: str = EDGE_LIST) -> None:
    """psp::save_graph (graph_io.hpp:21)."""
    eu, ev, ew, p = _edges(g)
    _lib.check(_lib.lib().psp_save_graph(g.n, len(eu), p(eu), p(ev), p(ew), os.fsencode(path),
                                         _format(fmt)))


def format_weight(w: float) -> str:
    """psp::format_weight (graph_io.hpp:25): shortest exact decimal."""
    buf = C.create_string_buffer(32)
    k = _lib.lib().psp_format_weight(float(w), buf)
    return buf.raw[:k].decode()


def random_pairs(n: int, count: int, seed: int, order: str = "cli"):
    """Seeded mt19937_64 pairs, rng() % n per endpoint.

    order="cli": v1 is drawn first, as tools/psp_main.cpp:108-120 does.
    order="tests": ref::random_pairs (tests/support/reference.hpp:80-91) as
    compiled by g++, which evaluates emplace_back's two rng() calls right to
    left, so v2 is the first draw."""
    v1 = np.empty(count, np.uint32)
    v2 = np.empty(count, np.uint32)
    _lib.lib().psp_random_pairs(n, count, seed, v1, v2)
    if order == "tests":
        return v2, v1
    if order != "cli":
        raise ValueError("order must be 'cli' or 'tests'")
    return v1, v2
