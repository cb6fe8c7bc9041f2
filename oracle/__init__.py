"""TEST INFRASTRUCTURE ONLY — CPU checkers for the GPU hot path.

Two ctypes front ends, both used exclusively by ``tests/``, by
``__graft_entry__.smoke()`` and by ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` arm — never by the product package
``paper_1503_07192_b200``:

* :class:`RefLib` — the UNMODIFIED reference library (``/root/reference/proj``)
  compiled by ``oracle/Makefile`` into ``oracle/_ref/libpspref.so`` and reached
  through ``oracle/ref_capi.cpp``.
* :class:`Oracle` — the plain-C restatement ``oracle/psp_oracle.c`` of the hot
  path (Phase 2 component APSP, Phase 3 boundary graph + Dijkstra rows, and
  Algorithm 2 queries), in the reference's f64 arithmetic.

The restatement is pinned against the reference build and against the golden
vectors of the reference's own tests (``tests/test_oracle_pin.py``).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libpspref.so")
ORACLE_SO = os.path.join(HERE, "_build", "libpsporacle.so")
SHIM_DIR = os.path.join(HERE, "_ref", "shim")
SHIM_TESTS = ("test_shortest_paths", "test_oracle", "test_query", "test_cluster")
REF_SRC = "/root/reference/proj"

_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")


def build(force: bool = False) -> None:
    """Compile the checkers (the reference part only where its sources exist)."""
    targets = ["oracle"]
    if os.path.isdir(REF_SRC):
        # the reference build and its own unit tests against the reference
        # and against the GPU shim (needs the product library built first)
        targets += ["ref", "shimtests"]
    args = ["make", "-s", "-j", "8", "-C", HERE] + (["-B"] if force else []) + targets
    subprocess.run(args, check=True)


# --------------------------------------------------------------- reference --
class RefError(RuntimeError):
    pass


class RefLib:
    """ctypes view of oracle/_ref/libpspref.so (the reference itself)."""

    _lib = None

    def __init__(self) -> None:
        if RefLib._lib is None:
            if not os.path.exists(REF_SO):
                raise FileNotFoundError(f"{REF_SO} missing: run `make -C oracle ref` where "
                                        f"{REF_SRC} exists")
            lib = C.CDLL(REF_SO)
            vp = C.c_void_p
            lib.ref_last_error.restype = C.c_char_p
            lib.ref_generate.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_int, C.c_double,
                                         C.c_double, C.c_uint64, C.POINTER(vp)]
            lib.ref_graph_from_edges.argtypes = [C.c_uint64, C.c_uint64, _u32p, _u32p, _f64p,
                                                 C.POINTER(vp)]
            lib.ref_graph_n.argtypes = [vp]
            lib.ref_graph_n.restype = C.c_uint64
            lib.ref_graph_m.argtypes = [vp]
            lib.ref_graph_m.restype = C.c_uint64
            lib.ref_graph_edges.argtypes = [vp, _u32p, _u32p, _f64p]
            lib.ref_graph_free.argtypes = [vp]
            lib.ref_oracle_free.argtypes = [vp]
            lib.ref_partition.argtypes = [vp, C.c_uint32, C.c_uint64, _u32p,
                                          C.POINTER(C.c_double)]
            lib.ref_apsp_dense.argtypes = [vp, C.c_uint64, _f64p]
            lib.ref_dijkstra.argtypes = [vp, C.c_uint32, _f64p]
            lib.ref_build_oracle.argtypes = [vp, C.c_uint32, C.c_uint32, C.c_uint64, _f64p,
                                             C.POINTER(vp)]
            lib.ref_oracle_info.argtypes = [vp, _u64p]
            lib.ref_oracle_ids.argtypes = [vp, _u32p, _u32p, _u64p, _u64p, _u32p, _u8p]
            lib.ref_oracle_component.argtypes = [vp, C.c_uint32, _f64p]
            lib.ref_oracle_boundary_rows.argtypes = [vp, C.c_uint32, _f64p]
            lib.ref_batch_query.argtypes = [vp, C.c_uint64, _u32p, _u32p, C.c_uint32, _f64p,
                                            C.c_void_p, C.POINTER(C.c_double)]
            lib.ref_sampled_build.argtypes = [vp, C.c_uint32, C.c_uint32, C.c_uint64,
                                              C.c_uint32, C.c_uint64, _f64p, _u64p]
            lib.ref_random_pairs.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, _u32p, _u32p]
            lib.ref_sampled_oracle.argtypes = [vp, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint32,
                                               C.c_uint64, _f64p, _u64p, _u32p, C.POINTER(vp)]
            lib.ref_oracle_assemble.argtypes = [C.c_uint64, C.c_uint32, _u32p, _u32p, _u8p, _u64p,
                                                _u64p, _u32p, C.POINTER(C.c_void_p),
                                                C.POINTER(C.c_void_p), C.POINTER(vp)]
            lib.ref_save_oracle.argtypes = [vp, C.c_char_p]
            lib.ref_load_oracle.argtypes = [C.c_char_p, C.POINTER(vp)]
            lib.ref_read_graph.argtypes = [C.c_char_p, C.c_uint64, C.c_int, C.c_char_p,
                                           C.POINTER(vp), C.POINTER(C.c_int),
                                           C.POINTER(C.c_uint64)]
            lib.ref_write_graph.argtypes = [vp, C.c_int, C.c_char_p, C.c_uint64,
                                            C.POINTER(C.c_uint64)]
            lib.ref_place_components.argtypes = [C.c_uint32, C.c_uint32, C.c_int, _u32p]
            lib.ref_routed_query.argtypes = [vp, C.c_uint32, C.c_int, C.c_uint32, C.c_uint32,
                                             C.c_uint64, _f64p]
            lib.ref_cluster_run_batch.argtypes = [vp, C.c_uint32, C.c_int, C.c_uint64, _u32p,
                                                  _u32p, _f64p, _u64p, C.POINTER(C.c_uint64)]
            lib.ref_simulate_build_schedule.argtypes = [C.c_uint32, C.c_uint32, _f64p, C.c_int,
                                                        _f64p, C.POINTER(C.c_double),
                                                        C.POINTER(C.c_double)]
            RefLib._lib = lib
        self.lib = RefLib._lib

    def _check(self, rc: int) -> None:
        if rc != 0:
            raise RefError(self.lib.ref_last_error().decode())

    def random_pairs(self, n: int, count: int, seed: int):
        """ref::random_pairs (tests/support/reference.hpp:80-91)."""
        v1 = np.empty(count, np.uint32)
        v2 = np.empty(count, np.uint32)
        self.lib.ref_random_pairs(n, count, seed, v1, v2)
        return v1, v2

    # graph text (include/psp/graph_io.hpp) -----------------------------
    def read_graph(self, text, fmt: int = 0, name: str = "<stream>"):
        """psp::read_graph: returns ("ok", RefGraph) or (kind, message, line)
        with kind "parse" | "graph" | "io" | "other"."""
        data = text.encode() if isinstance(text, str) else bytes(text)
        h, kind, line = C.c_void_p(), C.c_int(), C.c_uint64()
        rc = self.lib.ref_read_graph(data, len(data), fmt, name.encode(), C.byref(h),
                                     C.byref(kind), C.byref(line))
        if rc == 0:
            return "ok", RefGraph(self, h)
        kinds = {1: "parse", 2: "graph", 3: "io", 4: "other"}
        return kinds[kind.value], self.lib.ref_last_error().decode(), int(line.value)

    def write_graph(self, g: "RefGraph", fmt: int = 0) -> str:
        n = C.c_uint64()
        self._check(self.lib.ref_write_graph(g.h, fmt, None, 0, C.byref(n)))
        buf = C.create_string_buffer(max(n.value, 1))
        self._check(self.lib.ref_write_graph(g.h, fmt, buf, n.value, C.byref(n)))
        return buf.raw[: n.value].decode()

    # cluster layer (include/psp/placement.hpp, include/psp/cluster.hpp) ---
    def place_components(self, k: int, p: int, policy: int = 0) -> np.ndarray:
        owner = np.empty(max(k, 1), np.uint32)
        self._check(self.lib.ref_place_components(k, p, policy, owner))
        return owner[:k]

    def simulate_build_schedule(self, k: int, p: int, costs, policy: int = 0):
        costs = np.ascontiguousarray(costs, np.float64)
        wc = np.empty(max(p, 1), np.float64)
        mk, ml = C.c_double(), C.c_double()
        self._check(self.lib.ref_simulate_build_schedule(k, p, costs, policy, wc, C.byref(mk),
                                                         C.byref(ml)))
        return wc[:p].tolist(), mk.value, ml.value

    def load_oracle(self, path: str) -> "RefOracle":
        """psp::load_oracle on the reference."""
        h = C.c_void_p()
        self._check(self.lib.ref_load_oracle(os.fsencode(path), C.byref(h)))
        return RefOracle(self, h, np.zeros(7))

    # graphs ------------------------------------------------------------
    def generate(self, kind: str, rows: int, cols: int, weights=None, seed: int = 0) -> "RefGraph":
        """kind 'grid' | 'tri'; weights None (unit) or (lo, hi) uniform lattice."""
        h = C.c_void_p()
        unit = 1 if weights is None else 0
        lo, hi = (1.0, 1.0) if weights is None else weights
        self._check(self.lib.ref_generate(0 if kind == "grid" else 1, rows, cols, unit, lo, hi,
                                          seed, C.byref(h)))
        return RefGraph(self, h)

    def graph(self, n: int, eu, ev, ew) -> "RefGraph":
        eu = np.ascontiguousarray(eu, np.uint32)
        ev = np.ascontiguousarray(ev, np.uint32)
        ew = np.ascontiguousarray(ew, np.float64)
        h = C.c_void_p()
        self._check(self.lib.ref_graph_from_edges(n, len(eu), eu, ev, ew, C.byref(h)))
        return RefGraph(self, h)


class RefGraph:
    def __init__(self, ref: RefLib, h) -> None:
        self.ref, self.h = ref, h
        self.n = int(ref.lib.ref_graph_n(h))
        self.m = int(ref.lib.ref_graph_m(h))

    def __del__(self):
        try:
            self.ref.lib.ref_graph_free(self.h)
        except Exception:
            pass

    def edges(self):
        eu = np.empty(self.m, np.uint32)
        ev = np.empty(self.m, np.uint32)
        ew = np.empty(self.m, np.float64)
        self.ref._check(self.ref.lib.ref_graph_edges(self.h, eu, ev, ew))
        return eu, ev, ew

    def partition(self, k: int, seed: int = 0):
        a = np.empty(self.n, np.uint32)
        ms = C.c_double()
        self.ref._check(self.ref.lib.ref_partition(self.h, k, seed, a, C.byref(ms)))
        return a, ms.value

    def apsp_dense(self, block: int = 64) -> np.ndarray:
        out = np.empty(self.n * self.n, np.float64)
        self.ref._check(self.ref.lib.ref_apsp_dense(self.h, block, out))
        return out.reshape(self.n, self.n)

    def dijkstra(self, src: int) -> np.ndarray:
        out = np.empty(self.n, np.float64)
        self.ref._check(self.ref.lib.ref_dijkstra(self.h, src, out))
        return out

    def build_oracle(self, k: int, workers: int = 1, seed: int = 0) -> "RefOracle":
        stats = np.zeros(7, np.float64)
        h = C.c_void_p()
        self.ref._check(self.ref.lib.ref_build_oracle(self.h, k, workers, seed, stats, C.byref(h)))
        return RefOracle(self.ref, h, stats)

    def sampled_build(self, k: int, workers: int, rows: int, seed: int = 0, sample_seed: int = 1):
        times = np.zeros(4, np.float64)
        info = np.zeros(2, np.uint64)
        self.ref._check(self.ref.lib.ref_sampled_build(self.h, k, workers, seed, rows,
                                                       sample_seed, times, info))
        return dict(partition_ms=times[0], component_apsp_ms=times[1], bg_build_ms=times[2],
                    sampled_dijkstra_ms=times[3], rows=rows, b=int(info[0]),
                    bg_edges=int(info[1]))


    def sampled_oracle(self, k: int, workers: int, n_comps: int, seed: int = 0,
                       sample_seed: int = 1):
        """ref_sampled_oracle: the reference's Phases 1-2 in full, the
        boundary graph in full, and the reference's Dijkstra rows for the
        boundary vertices of `n_comps` seeded components only. Returns the
        (partial) RefOracle, the sampled components and the phase times."""
        times = np.zeros(4, np.float64)
        info = np.zeros(3, np.uint64)
        comps = np.zeros(max(1, min(n_comps, k)), np.uint32)
        h = C.c_void_p()
        self.ref._check(self.ref.lib.ref_sampled_oracle(self.h, k, workers, seed, n_comps,
                                                        sample_seed, times, info, comps,
                                                        C.byref(h)))
        ro = RefOracle(self.ref, h, np.zeros(7))
        return ro, comps, dict(partition_ms=times[0], component_apsp_ms=times[1],
                               bg_build_ms=times[2], sampled_rows_ms=times[3],
                               rows=int(info[2]), b=int(info[0]), bg_edges=int(info[1]))


def assemble_oracle(ref: "RefLib", n, k, perm, assign, flags, comp_off, bnd_off, bvert,
                    ct: list, bt: list) -> "RefOracle":
    """ref_oracle_assemble: a psp::Oracle from plain arrays (bt[c] / ct[c]
    None = component not sampled) so that the reference's batch_query runs on
    it over pairs that touch sampled components only."""
    ctp = (C.c_void_p * k)(*[(t.ctypes.data if t is not None else None) for t in ct])
    btp = (C.c_void_p * k)(*[(t.ctypes.data if t is not None else None) for t in bt])
    h = C.c_void_p()
    ref._check(ref.lib.ref_oracle_assemble(
        n, k, np.ascontiguousarray(perm, np.uint32), np.ascontiguousarray(assign, np.uint32),
        np.ascontiguousarray(flags, np.uint8), np.ascontiguousarray(comp_off, np.uint64),
        np.ascontiguousarray(bnd_off, np.uint64), np.ascontiguousarray(bvert, np.uint32),
        ctp, btp, C.byref(h)))
    ro = RefOracle(ref, h, np.zeros(7))
    ro._keep = (ct, bt)
    return ro


STAT_KEYS = ("partition_ms", "component_apsp_ms", "boundary_ms", "boundary_total", "bg_edges",
             "stored_entries", "peak_table_entries_per_worker")


class RefOracle:
    def __init__(self, ref: RefLib, h, stats) -> None:
        self.ref, self.h = ref, h
        self.stats = dict(zip(STAT_KEYS, stats.tolist()))
        info = np.zeros(3, np.uint64)
        ref.lib.ref_oracle_info(h, info)
        self.n, self.k, self.b = (int(x) for x in info)
        self.permutation = np.empty(self.n, np.uint32)
        self.assignment = np.empty(self.n, np.uint32)  # reordered id space
        self.boundary_flags = np.empty(self.n, np.uint8)
        self.component_offset = np.empty(self.k + 1, np.uint64)
        self.boundary_offset = np.empty(self.k + 1, np.uint64)
        self.boundary_vertex = np.empty(max(self.b, 1), np.uint32)
        ref.lib.ref_oracle_ids(h, self.permutation, self.assignment, self.component_offset,
                               self.boundary_offset, self.boundary_vertex, self.boundary_flags)
        self.boundary_vertex = self.boundary_vertex[: self.b]

    def __del__(self):
        try:
            self.ref.lib.ref_oracle_free(self.h)
        except Exception:
            pass

    def component_size(self, c: int) -> int:
        return int(self.component_offset[c + 1] - self.component_offset[c])

    def boundary_size(self, c: int) -> int:
        return int(self.boundary_offset[c + 1] - self.boundary_offset[c])

    def save(self, path: str) -> None:
        """psp::save_oracle on the reference."""
        self.ref._check(self.ref.lib.ref_save_oracle(self.h, os.fsencode(path)))

    def component_table(self, c: int) -> np.ndarray:
        s = self.component_size(c)
        out = np.empty(s * s, np.float64)
        self.ref.lib.ref_oracle_component(self.h, c, out)
        return out.reshape(s, s)

    def boundary_rows(self, c: int) -> np.ndarray:
        r = self.boundary_size(c)
        out = np.empty(max(r * self.b, 1), np.float64)
        self.ref.lib.ref_oracle_boundary_rows(self.h, c, out)
        return out[: r * self.b].reshape(r, self.b)

    def routed_query(self, p: int, v1: int, v2: int, query_id: int = 0, policy: int = 0) -> dict:
        """psp::routed_query (src/cluster.cpp:49-74) under place_components(k, p)."""
        out = np.empty(15, np.float64)
        self.ref._check(self.ref.lib.ref_routed_query(self.h, p, policy, v1, v2, query_id, out))
        keys = ("distance", "minplus_ops", "b1", "b2", "same_component", "transfer_entries",
                "executed_on", "column_owner", "has_transfer", "src_worker", "dst_worker",
                "entries", "bytes", "overlap_cost", "serial_cost")
        return dict(zip(keys, out.tolist()))

    def cluster_run_batch(self, p: int, v1, v2, policy: int = 0):
        """psp::ClusterSim::run_batch (src/cluster.cpp:225-231): distances and
        the ledger rows (query_id, src_worker, dst_worker, entries, bytes)."""
        v1 = np.ascontiguousarray(v1, np.uint32)
        v2 = np.ascontiguousarray(v2, np.uint32)
        dist = np.empty(len(v1), np.float64)
        rec = np.empty(max(5 * len(v1), 5), np.uint64)
        nrec = C.c_uint64()
        self.ref._check(self.ref.lib.ref_cluster_run_batch(self.h, p, policy, len(v1), v1, v2,
                                                           dist, rec, C.byref(nrec)))
        return dist, rec[: 5 * nrec.value].reshape(-1, 5)

    def batch_query(self, v1, v2, workers: int = 1, with_ops: bool = False):
        v1 = np.ascontiguousarray(v1, np.uint32)
        v2 = np.ascontiguousarray(v2, np.uint32)
        dist = np.empty(len(v1), np.float64)
        ops = np.empty(len(v1), np.uint64) if with_ops else None
        ms = C.c_double()
        self.ref._check(self.ref.lib.ref_batch_query(
            self.h, len(v1), v1, v2, workers, dist,
            ops.ctypes.data_as(C.c_void_p) if ops is not None else None, C.byref(ms)))
        self.last_query_ms = ms.value
        return (dist, ops) if with_ops else dist


# ----------------------------------------------------------- restatement --
class Oracle:
    """The plain-C restatement (oracle/psp_oracle.c) built on a given partition.

    Inputs are the ORIGINAL graph edges plus a partition given as the
    original->reordered permutation, the reordered assignment and reordered
    boundary flags (exactly what psp::reorder_vertices produces).
    """

    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            if not os.path.exists(ORACLE_SO):
                build()
            lib = C.CDLL(ORACLE_SO)
            lib.pso_apsp_dense.argtypes = [C.c_uint64, _u64p, _u32p, _f64p, C.c_uint64, _f64p]
            lib.pso_dijkstra.argtypes = [C.c_uint64, _u64p, _u32p, _f64p, C.c_uint32, _f64p]
            lib.pso_min_plus_combine.argtypes = [C.c_uint64, _f64p, _f64p]
            lib.pso_min_plus_combine.restype = C.c_double
            lib.pso_build.argtypes = [C.c_uint64, _u64p, _u32p, _f64p, C.c_uint32, _u32p, _u32p,
                                      _u8p]
            lib.pso_build.restype = C.c_void_p
            lib.pso_free.argtypes = [C.c_void_p]
            lib.pso_info.argtypes = [C.c_void_p, _u64p]
            lib.pso_offsets.argtypes = [C.c_void_p, _u64p, _u64p]
            lib.pso_component_table.argtypes = [C.c_void_p, C.c_uint32]
            lib.pso_component_table.restype = C.POINTER(C.c_double)
            lib.pso_boundary_rows.argtypes = [C.c_void_p, C.c_uint32]
            lib.pso_boundary_rows.restype = C.POINTER(C.c_double)
            lib.pso_batch_query.argtypes = [C.c_void_p, C.c_uint64, _u32p, _u32p, _f64p,
                                            C.c_void_p]
            lib.pso_batch_query.restype = C.c_uint64
            cls._lib = lib
        return cls._lib

    def __init__(self, n, eu, ev, ew, k, perm, assign_reordered, flags_reordered):
        lib = self.lib()
        off, to, w = reordered_csr(n, eu, ev, ew, perm)
        self.h = lib.pso_build(n, off, to, w, k, np.ascontiguousarray(perm, np.uint32),
                               np.ascontiguousarray(assign_reordered, np.uint32),
                               np.ascontiguousarray(flags_reordered, np.uint8))
        info = np.zeros(5, np.uint64)
        lib.pso_info(self.h, info)
        self.n, self.k, self.b, self.bg_edges, self.stored_entries = (int(x) for x in info)
        self.component_offset = np.empty(self.k + 1, np.uint64)
        self.boundary_offset = np.empty(self.k + 1, np.uint64)
        lib.pso_offsets(self.h, self.component_offset, self.boundary_offset)

    def __del__(self):
        try:
            self.lib().pso_free(self.h)
        except Exception:
            pass

    def component_table(self, c: int) -> np.ndarray:
        s = int(self.component_offset[c + 1] - self.component_offset[c])
        p = self.lib().pso_component_table(self.h, c)
        return np.ctypeslib.as_array(p, shape=(max(s * s, 1),))[: s * s].reshape(s, s).copy()

    def boundary_rows(self, c: int) -> np.ndarray:
        r = int(self.boundary_offset[c + 1] - self.boundary_offset[c])
        p = self.lib().pso_boundary_rows(self.h, c)
        return np.ctypeslib.as_array(p, shape=(max(r * self.b, 1),))[: r * self.b].reshape(
            r, self.b).copy()

    def batch_query(self, v1, v2, with_ops: bool = False):
        v1 = np.ascontiguousarray(v1, np.uint32)
        v2 = np.ascontiguousarray(v2, np.uint32)
        dist = np.empty(len(v1), np.float64)
        ops = np.empty(len(v1), np.uint64) if with_ops else None
        bad = self.lib().pso_batch_query(self.h, len(v1), v1, v2, dist,
                                         ops.ctypes.data_as(C.c_void_p) if ops is not None
                                         else None)
        if bad:
            raise ValueError("query: vertex id out of range")
        return (dist, ops) if with_ops else dist


def csr(n, eu, ev, ew):
    """Sorted symmetric CSR, as psp::Graph builds it (src/graph.cpp:19-56)."""
    eu = np.asarray(eu, np.int64)
    ev = np.asarray(ev, np.int64)
    ew = np.asarray(ew, np.float64)
    src = np.concatenate([eu, ev])
    dst = np.concatenate([ev, eu])
    w = np.concatenate([ew, ew])
    order = np.lexsort((dst, src))
    src, dst, w = src[order], dst[order], w[order]
    off = np.zeros(n + 1, np.uint64)
    np.add.at(off, src + 1, 1)
    off = np.cumsum(off).astype(np.uint64)
    return off, dst.astype(np.uint32), np.ascontiguousarray(w)


def reordered_csr(n, eu, ev, ew, perm):
    perm = np.asarray(perm, np.int64)
    return csr(n, perm[np.asarray(eu, np.int64)], perm[np.asarray(ev, np.int64)], ew)


def apsp_dense(n, eu, ev, ew, block: int = 64) -> np.ndarray:
    off, to, w = csr(n, eu, ev, ew)
    out = np.empty(max(n * n, 1), np.float64)
    if Oracle.lib().pso_apsp_dense(n, off, to, w, block, out) != 0:
        raise ValueError("apsp_dense: block size must be positive")
    return out[: n * n].reshape(n, n)


def dijkstra(n, eu, ev, ew, src: int) -> np.ndarray:
    off, to, w = csr(n, eu, ev, ew)
    out = np.empty(n, np.float64)
    Oracle.lib().pso_dijkstra(n, off, to, w, src, out)
    return out


def min_plus_combine(a, b) -> float:
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    if len(a) != len(b):
        raise ValueError("min_plus_combine: length mismatch")
    return float(Oracle.lib().pso_min_plus_combine(len(a), a, b))

