"""Distributed query mode: the reference's placement + cluster layer
(include/psp/placement.hpp, include/psp/cluster.hpp, src/cluster.cpp) with
the simulated workers replaced by GPU ranks.

* :func:`place_components` -- psp::place_components (placement.cpp:7-33),
  computed by the C-ABI.
* :class:`TransferLedger` / :class:`TransferRecord` -- the reference's
  append-only transfer log and its CSV (cluster.cpp:11-47).
* :func:`routed_query` -- psp::routed_query (cluster.cpp:49-74): the distance
  from the device oracle plus the routing facts and the two cost models.
* :class:`RoutedOracle` -- the ClusterSim analogue (cluster.hpp:79-109) on
  real GPUs: every rank keeps only its components' tables
  (psp_gpu_shard_create), a batch executes each query at owner(C1) and reads
  col2 from owner(C2) over NVLink (psp_gpu_routed_query_batch). Collective:
  every rank of the context constructs it and calls run_batch together.
* :func:`simulate_build_schedule` -- the Phase-3 imbalance study
  (cluster.cpp:233-251), pure host arithmetic.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import threading

import numpy as np

from . import _lib

ROUND_ROBIN = "round_robin"
PAIRS_PER_GPU = "pairs_per_gpu"
_POLICY = {ROUND_ROBIN: _lib.PLACE_ROUND_ROBIN, PAIRS_PER_GPU: _lib.PLACE_PAIRS_PER_GPU}


@dataclasses.dataclass
class Placement:
    """psp::Placement (placement.hpp:19-25)."""
    p: int
    owner: np.ndarray                      # [k] uint32
    components_of: list                    # [p] lists of component ids


def place_components(k: int, p: int, policy: str = ROUND_ROBIN) -> Placement:
    if policy not in _POLICY:
        raise ValueError(f"place_components: unknown policy {policy!r}")
    owner = np.empty(max(k, 1), np.uint32)
    _lib.check(_lib.lib().psp_place_components(k, p, _POLICY[policy], owner))
    owner = owner[:k]
    comps = [[] for _ in range(p)]
    for c, w in enumerate(owner.tolist()):
        comps[w].append(c)
    return Placement(p, owner, comps)


@dataclasses.dataclass(frozen=True)
class TransferRecord:
    """psp::TransferRecord (cluster.hpp:22-31): col2 shipped from
    src_worker = owner(C2) to dst_worker = owner(C1)."""
    query_id: int
    src_worker: int
    dst_worker: int
    entries: int
    bytes: int


class TransferLedger:
    """psp::TransferLedger (cluster.hpp:35-50): thread-safe append-only log.

    Stored columnar (rows of query_id, src_worker, dst_worker, entries,
    bytes as uint64) because a routed batch appends up to one record per
    query; records() materialises TransferRecord objects on demand."""

    _EMPTY = np.empty((0, 5), np.uint64)

    def __init__(self):
        self._mu = threading.Lock()
        self._chunks: list = []  # (N, 5) arrays, or routed batches still to expand

    @staticmethod
    def _rows(chunk) -> np.ndarray:
        if isinstance(chunk, np.ndarray):
            return chunk
        base, ex, co, ent = chunk  # a routed batch: a record iff owner(C1) != owner(C2)
        cross = np.flatnonzero(ex != co)
        rows = np.empty((len(cross), 5), np.uint64)
        rows[:, 0] = base + cross
        rows[:, 1] = co[cross]
        rows[:, 2] = ex[cross]
        rows[:, 3] = ent[cross]  # B2 (src/cluster.cpp:83)
        rows[:, 4] = 8 * rows[:, 3]
        return rows

    def _extend_routed(self, base: int, ex, co, ent) -> None:
        """Append a routed batch's records without expanding them yet (a
        batch can carry one record per query; expansion is deferred to the
        first read)."""
        with self._mu:
            self._chunks.append((base, ex, co, ent))

    def record(self, rec: TransferRecord) -> None:
        row = np.array([[rec.query_id, rec.src_worker, rec.dst_worker, rec.entries, rec.bytes]],
                       np.uint64)
        with self._mu:
            self._chunks.append(row)

    def extend_rows(self, rows: np.ndarray) -> None:
        """Append an (N, 5) array of records."""
        rows = np.ascontiguousarray(rows, np.uint64).reshape(-1, 5)
        if len(rows):
            with self._mu:
                self._chunks.append(rows)

    def as_array(self) -> np.ndarray:
        with self._mu:
            return self._flat().copy()

    def _flat(self) -> np.ndarray:  # caller holds the lock
        if not self._chunks:
            return self._EMPTY
        if len(self._chunks) > 1 or not isinstance(self._chunks[0], np.ndarray):
            self._chunks = [np.concatenate([self._rows(c) for c in self._chunks])]
        return self._chunks[0]

    def records(self) -> list[TransferRecord]:
        return [TransferRecord(*map(int, r)) for r in self.as_array()]

    def size(self) -> int:
        with self._mu:
            return len(self._flat())

    def total_entries(self) -> int:
        with self._mu:
            return int(self._flat()[:, 3].sum())

    def total_bytes(self) -> int:
        with self._mu:
            return int(self._flat()[:, 4].sum())

    def write_csv(self, out) -> None:
        """"query_id,src_worker,dst_worker,entries,bytes", one row each
        (cluster.cpp:40-47)."""
        rows = self.as_array()
        out.write("query_id,src_worker,dst_worker,entries,bytes\n")
        if len(rows):
            out.write("\n".join(",".join(map(str, r)) for r in rows.tolist()) + "\n")


@dataclasses.dataclass
class QueryResult:
    """psp::QueryResult + QueryStats (query.hpp:15-33)."""
    distance: float
    minplus_ops: int
    boundary_size_1: int
    boundary_size_2: int
    same_component: bool
    transfer_entries: int = 0


@dataclasses.dataclass
class RoutedQueryResult:
    """psp::RoutedQueryResult (cluster.hpp:55-64)."""
    result: QueryResult
    executed_on: int
    column_owner: int
    transfer: TransferRecord | None
    overlap_cost: float  # max(B1*B2, transfer_entries) + B2
    serial_cost: float   # B1*B2 + transfer_entries + B2


def _components(oracle, v1, v2):
    perm, assign = oracle.permutation, oracle.assignment
    return assign[perm[np.asarray(v1, np.int64)]], assign[perm[np.asarray(v2, np.int64)]]


def routed_query(oracle, placement: Placement, v1: int, v2: int,
                 query_id: int = 0) -> RoutedQueryResult:
    """psp::routed_query (cluster.cpp:49-74) over a replicated GpuOracle."""
    d, ops = oracle.query(v1, v2)  # raises ValueError on ids >= n (query.cpp:30)
    c1, c2 = (int(x[0]) for x in _components(oracle, [v1], [v2]))
    b1, b2 = oracle.boundary_size(c1), oracle.boundary_size(c2)
    ex, co = int(placement.owner[c1]), int(placement.owner[c2])
    moved = b2 if ex != co else 0
    rec = TransferRecord(query_id, co, ex, b2, 8 * b2) if ex != co else None
    qr = QueryResult(d, ops, b1, b2, c1 == c2, moved)
    return RoutedQueryResult(qr, ex, co, rec, float(max(b1 * b2, moved) + b2),
                             float(b1 * b2 + moved + b2))


class RoutedOracle:
    """ClusterSim on GPUs (cluster.hpp:79-109, cluster.cpp:118-231).

    Built from a replicated GpuOracle on a context of `world` ranks with the
    placement's p == world; afterwards this rank holds only its components'
    tables and the source oracle may be closed. run_batch is collective: every
    rank calls it with its own pairs (possibly none); the ledger records the
    transfers of the pairs THIS rank submitted, numbered by a running query id
    like ClusterSim's next_query_id_ (cluster.cpp:213)."""

    def __init__(self, oracle, placement: Placement):
        if len(placement.owner) != oracle.k:
            raise ValueError("ClusterSim: placement does not cover the oracle")
        if placement.p != oracle.ctx.world:
            raise ValueError("RoutedOracle: placement.p must equal the context's world size")
        self.ctx, self.placement = oracle.ctx, placement
        self.n, self.k, self.b = oracle.n, oracle.k, oracle.b
        self.permutation = oracle.permutation
        self.assignment = oracle.assignment
        self.boundary_offset = oracle.boundary_offset
        self._ledger = TransferLedger()
        self._next_query_id = 0
        self.last_stats: dict | None = None
        h = C.c_void_p()
        owner = np.ascontiguousarray(placement.owner, np.uint32)
        _lib.check(_lib.lib().psp_gpu_shard_create(oracle.h, owner, C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            h, self.h = self.h, None
            _lib.check(_lib.lib().psp_gpu_shard_free(h))

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def device_bytes(self) -> int:
        out = C.c_uint64()
        _lib.check(_lib.lib().psp_gpu_shard_bytes(self.h, C.byref(out)))
        return int(out.value)

    def ledger(self) -> TransferLedger:
        return self._ledger

    def run_batch(self, v1, v2, with_routing: bool = False):
        """Distances of this rank's pairs (f64, +inf unreachable), computed
        at owner(C1) with col2 from owner(C2). With with_routing, also
        returns (executed_on, column_owner, transfer_entries) arrays."""
        v1 = np.ascontiguousarray(v1, np.uint32)
        v2 = np.ascontiguousarray(v2, np.uint32)
        if v1.shape != v2.shape:
            raise ValueError("run_batch: v1 and v2 differ in length")
        n = len(v1)
        dist = np.empty(n, np.float64)
        ex = np.empty(n, np.uint32)
        co = np.empty(n, np.uint32)
        ent = np.empty(n, np.uint32)
        st = _lib.RoutedStats()
        p = lambda a: a.ctypes.data_as(C.c_void_p)
        _lib.check(_lib.lib().psp_gpu_routed_query_batch(self.h, n, p(v1), p(v2), p(dist), p(ex),
                                                        p(co), p(ent), C.byref(st)))
        self.last_stats = st.as_dict()
        self._ledger._extend_routed(self._next_query_id, ex, co, ent)
        self._next_query_id += n
        return (dist, ex, co, ent) if with_routing else dist

    def run_query(self, v1: int, v2: int) -> float:
        return float(self.run_batch([v1], [v2])[0])


@dataclasses.dataclass
class ScheduleProfile:
    """psp::ScheduleProfile (cluster.hpp:113-119)."""
    worker_cost: list
    makespan: float
    mean_load: float


def simulate_build_schedule(k: int, p: int, component_costs,
                            policy: str = ROUND_ROBIN) -> ScheduleProfile:
    """psp::simulate_build_schedule (cluster.cpp:233-251)."""
    costs = [float(x) for x in component_costs]
    if len(costs) != k:
        raise ValueError("simulate_build_schedule: need one cost per component")
    pl = place_components(k, p, policy)
    worker = [0.0] * p
    total = 0.0
    for c in range(k):
        worker[int(pl.owner[c])] += costs[c]
        total += costs[c]
    return ScheduleProfile(worker, max(worker), total / p)
