"""Pin the CPU oracle (oracle/psp_oracle.c) before trusting it.

1. Golden vectors spelled out in the reference's own tests (file:line cited).
2. The committed fixtures tests/golden/*.npz, produced by the UNMODIFIED
   reference build (tests/golden/make_golden.py).
3. The live reference build (oracle/_ref) on further graphs, when present.
"""
from __future__ import annotations

import hashlib
import math

import numpy as np
import pytest

import oracle
from conftest import graph_of

INF = math.inf


def restated(case):
    """Oracle restatement built on the fixture's (reference) partition."""
    n = int(case["n"])
    perm = case["permutation"]
    assign_r = np.empty(n, np.uint32)
    assign_r[perm] = case["assignment"]
    # boundary flags in reordered space: boundary-first prefixes of each range
    flags = np.zeros(n, np.uint8)
    co, bo = case["component_offset"], case["boundary_offset"]
    for c in range(int(case["k"])):
        flags[int(co[c]): int(co[c]) + int(bo[c + 1] - bo[c])] = 1
    return oracle.Oracle(n, case["eu"], case["ev"], case["ew"], int(case["k"]), perm, assign_r,
                         flags)


# ---------------------------------------------------------- 1. golden -----
def test_grid2x3_every_table_spelled_out(golden_small):
    # tests/test_oracle.cpp:28-79
    case = golden_small["grid2x3_k2"]
    assert case["permutation"].tolist() == [2, 0, 3, 1, 4, 5]
    assert case["component_offset"].tolist() == [0, 3, 6]
    assert case["boundary_offset"].tolist() == [0, 2, 4]
    assert case["boundary_vertex"].tolist() == [0, 1, 3, 4]
    path = [0, 2, 1, 2, 0, 1, 1, 1, 0]
    o = restated(case)
    assert o.component_table(0).ravel().tolist() == path
    assert o.component_table(1).ravel().tolist() == path
    assert o.boundary_rows(0).ravel().tolist() == [0, 2, 1, 1, 2, 0, 3, 1]
    assert o.boundary_rows(1).ravel().tolist() == [1, 3, 0, 2, 1, 1, 2, 0]
    assert o.stored_entries == 34 and o.bg_edges == 5 and o.b == 4
    assert int(case["stored_entries"]) == 34 and int(case["bg_edges"]) == 5


def test_query_golden_vectors(golden_small):
    # tests/test_query.cpp:30-62 (0->5 = 3, ops 6), :64-89 (escape route = 5)
    o = restated(golden_small["grid2x3_k2"])
    d, ops = o.batch_query([0], [5], with_ops=True)
    assert d[0] == 3.0 and ops[0] == 6
    o8 = restated(golden_small["cycle8_k2_s4"])
    d, _ = o8.batch_query([2, 3], [5, 3], with_ops=True)
    assert d.tolist() == [5.0, 0.0]
    # tests/test_query.cpp:155-164: isolated vertices -> INF with 0 ops
    oi = restated(golden_small["isolated2_k2"])
    d, ops = oi.batch_query([0, 0], [1, 0], with_ops=True)
    assert d[0] == INF and ops[0] == 0 and d[1] == 0.0


def test_query_out_of_range_raises(golden_small):
    o = restated(golden_small["grid2x3_k2"])
    with pytest.raises(ValueError):
        o.batch_query([0], [6])


def test_dijkstra_and_min_plus_goldens():
    # tests/test_shortest_paths.cpp:14-20 on the 2x3 unit grid
    eu, ev = [0, 1, 3, 4, 0, 1, 2], [1, 2, 4, 5, 3, 4, 5]
    ew = [1.0] * 7
    assert oracle.dijkstra(6, eu, ev, ew, 0).tolist() == [0, 1, 2, 1, 2, 3]
    assert oracle.dijkstra(6, eu, ev, ew, 4).tolist() == [2, 1, 2, 1, 0, 1]
    # tests/test_shortest_paths.cpp:22-29
    d = oracle.dijkstra(5, [0, 2, 3], [1, 3, 4], [2.5, 1.0, 1.0], 0)
    assert d.tolist() == [0, 2.5, INF, INF, INF]
    # tests/test_shortest_paths.cpp:85-105
    assert oracle.min_plus_combine([3.0, 1.0, 8.0], [2.0, 5.0, 0.5]) == 5.0
    assert oracle.min_plus_combine([], []) == INF
    assert oracle.min_plus_combine([INF, 4.0], [1.0, INF]) == INF
    assert oracle.min_plus_combine([INF, 4.0], [1.0, 2.0]) == 6.0
    with pytest.raises(ValueError):
        oracle.min_plus_combine([1.0, 2.0, 3.0], [1.0])
    with pytest.raises(ValueError):
        oracle.apsp_dense(3, [0], [1], [1.0], block=0)


# --------------------------------------------------------- 2. fixtures ----
@pytest.mark.parametrize("name", ["grid2x3_k2", "grid2x3_k1", "cycle8_k2_s4", "two_squares_k2",
                                  "isolated2_k2", "grid16_k4", "grid16_k8_lattice", "tri9_k6",
                                  "grid10_k2", "tri20_k20_w0", "grid32_k32_unit"])
def test_restatement_matches_reference_fixtures(golden_small, name):
    case = golden_small[name]
    o = restated(case)
    k = int(case["k"])
    assert o.b == int(case["b"])
    assert o.bg_edges == int(case["bg_edges"])
    assert o.stored_entries == int(case["stored_entries"])
    h = hashlib.sha256()
    for c in range(k):
        ct, bt = o.component_table(c), o.boundary_rows(c)
        assert np.array_equal(ct, case[f"ct{c}"]), f"component {c}"
        assert np.array_equal(bt, case[f"bt{c}"]), f"boundary rows {c}"
        h.update(ct.tobytes())
        h.update(bt.tobytes())
    assert h.digest() == case["tables_sha256"].tobytes()
    d, ops = o.batch_query(case["q_v1"], case["q_v2"], with_ops=True)
    assert np.array_equal(d, case["q_dist"])
    assert np.array_equal(ops, case["q_ops"])


def test_restatement_matches_cfg1_fixture(golden_cfg1):
    case = golden_cfg1
    o = restated(case)
    h = hashlib.sha256()
    for c in range(int(case["k"])):
        h.update(o.component_table(c).tobytes())
        h.update(o.boundary_rows(c).tobytes())
    assert h.digest() == case["tables_sha256"].tobytes()
    d, ops = o.batch_query(case["q_v1"], case["q_v2"], with_ops=True)
    assert np.array_equal(d, case["q_dist"]) and np.array_equal(ops, case["q_ops"])


def test_fixture_queries_equal_truth(golden_small):
    # the fixtures themselves agree with plain Dijkstra on the original graph
    for name in ("tri20_k20_w0", "grid16_k8_lattice", "cycle8_k2_s4"):
        case = golden_small[name]
        n = int(case["n"])
        for v1, v2, d in list(zip(case["q_v1"], case["q_v2"], case["q_dist"]))[:60]:
            truth = oracle.dijkstra(n, case["eu"], case["ev"], case["ew"], int(v1))
            assert truth[int(v2)] == d


# ---------------------------------------------------- 3. live reference --
@pytest.mark.parametrize("kind,rows,cols,w,gseed,k", [
    ("grid", 12, 11, (0.25, 2.0), 5, 5),
    ("tri", 15, 13, (1.0, 9.0), 3, 7),
    ("grid", 30, 30, (1, 1025), 2, 30),
])
def test_restatement_matches_live_reference(ref, kind, rows, cols, w, gseed, k):
    rg = ref.generate(kind, rows, cols, w, gseed)
    ro = rg.build_oracle(k, 1, 0)
    eu, ev, ew = rg.edges()
    o = oracle.Oracle(rg.n, eu, ev, ew, k, ro.permutation, ro.assignment, ro.boundary_flags)
    for c in range(k):
        assert np.array_equal(o.component_table(c), ro.component_table(c))
        assert np.array_equal(o.boundary_rows(c), ro.boundary_rows(c))
    assert o.bg_edges == int(ro.stats["bg_edges"])
    v1, v2 = ref.random_pairs(rg.n, 2000, 11)
    d1, o1 = o.batch_query(v1, v2, with_ops=True)
    d2, o2 = ro.batch_query(v1, v2, 1, with_ops=True)
    assert np.array_equal(d1, d2) and np.array_equal(o1, o2)


def test_apsp_dense_matches_reference(ref):
    # tests/test_shortest_paths.cpp:55-74: blocked FW, block-size invariance
    rg = ref.generate("tri", 6, 7, (0.5, 5.0), 23)
    eu, ev, ew = rg.edges()
    want = rg.apsp_dense(64)
    for bs in (1, 3, 41, 64, 4096):
        assert np.array_equal(oracle.apsp_dense(rg.n, eu, ev, ew, bs), want)
