"""Host-side logic of the product library (no GPU needed): graph
validation, generators, the restated partitioner and the C-ABI surface."""
from __future__ import annotations

import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_1503_07192_b200 as P
from paper_1503_07192_b200 import _lib
from conftest import GOLDEN, ROOT, graph_of


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "psp_gpu.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(psp_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), s
    # and the Python binding covers exactly that surface
    assert set(syms) == set(_lib.SIGNATURES)
    assert L.psp_gpu_abi_version() == 5


def test_no_gpu_fails_loudly_or_works():
    # Without a device the context must fail with PSP_ECUDA/EINVAL, never
    # fall back to the CPU.
    L = _lib.lib()
    if L.psp_gpu_device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(P.PspError) as ei:
        P.Context(0)
    assert ei.value.status in (_lib.PSP_ECUDA, _lib.PSP_EINVAL)


def test_random_pairs_stream_matches_reference():
    # ref::random_pairs (tests/support/reference.hpp:86-88) evaluates
    # emplace_back(rng() % n, rng() % n) right to left under g++, so its v2 is
    # the first draw; the CLI's random_pairs (tools/psp_main.cpp:113-117)
    # draws v1 first. psp_random_pairs follows the CLI; order="tests" swaps.
    z = np.load(os.path.join(GOLDEN, "random_pairs_n1000_s123.npz"))
    v1, v2 = P.random_pairs(1000, 16, 123)
    assert np.array_equal(v2, z["v1"]) and np.array_equal(v1, z["v2"])
    t1, t2 = P.random_pairs(1000, 16, 123, order="tests")
    assert np.array_equal(t1, z["v1"]) and np.array_equal(t2, z["v2"])


@pytest.mark.parametrize("kind,rows,cols,w,seed", [
    ("grid", 64, 64, (1, 1025), 1), ("grid", 2, 3, None, 0), ("tri", 9, 9, (1.0, 3.0), 4),
    ("tri", 20, 20, (0.0, 1024.0), 3), ("grid", 16, 16, (0.5, 2.0), 9)])
def test_generators_match_reference(ref, kind, rows, cols, w, seed):
    g = (P.generate_grid if kind == "grid" else P.generate_triangulated_grid)(rows, cols, w, seed)
    eu, ev, ew = ref.generate(kind, rows, cols, w, seed).edges()
    a, b = np.minimum(g.eu, g.ev), np.maximum(g.eu, g.ev)
    o = np.lexsort((b, a))
    assert np.array_equal(a[o], eu) and np.array_equal(b[o], ev) and np.array_equal(g.ew[o], ew)


def test_generator_argument_errors():
    with pytest.raises(ValueError):
        P.generate_grid(0, 3)
    with pytest.raises(ValueError):
        P.generate_grid(3, 3, (2.0, 1.0))


@pytest.mark.parametrize("name", ["grid2x3_k2", "cycle8_k2_s4", "two_squares_k2", "isolated2_k2",
                                  "grid16_k4", "grid16_k8_lattice", "tri9_k6", "grid10_k2",
                                  "tri20_k20_w0", "grid32_k32_unit"])
def test_partition_matches_reference_fixtures(golden_small, name):
    case = golden_small[name]
    g = graph_of(case)
    a = P.partition_graph(g, int(case["k"]), int(case["seed"]), threads=4)
    assert np.array_equal(a, case["assignment"])


def test_partition_cfg1_fixture(golden_cfg1):
    g = graph_of(golden_cfg1)
    for threads in (1, 8):  # worker count never changes the result
        a = P.partition_graph(g, 16, 0, threads=threads)
        assert np.array_equal(a, golden_cfg1["assignment"])


@pytest.mark.parametrize("kind,rows,cols,w,gseed,k,seed", [
    ("grid", 40, 40, None, 0, 40, 0), ("tri", 25, 31, (1.0, 4.0), 2, 17, 3),
    ("grid", 33, 47, (1, 1025), 5, 64, 9), ("tri", 50, 50, (0.0, 1024.0), 1, 50, 1),
    ("grid", 7, 7, None, 0, 49, 0),  # k = n: every vertex its own component
])
def test_partition_matches_live_reference(ref, kind, rows, cols, w, gseed, k, seed):
    rg = ref.generate(kind, rows, cols, w, gseed)
    want, _ = rg.partition(k, seed)
    eu, ev, ew = rg.edges()
    got = P.partition_graph(P.Graph(rg.n, eu, ev, ew), k, seed, threads=8)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("case", ["permuted_grid", "permuted_tri", "delaunay", "delaunay_pieces"])
def test_partition_scrambled_ids_match_reference(ref, case):
    """Ids with no locality (the partitioner relabels internally in BFS
    order; every id-order rule must still be the reference's)."""
    rng = np.random.default_rng(11)
    if case.startswith("permuted"):
        rg = ref.generate("grid" if case == "permuted_grid" else "tri", 30, 37, (1.0, 9.0), 4)
        eu, ev, ew = rg.edges()
        n = rg.n
        perm = rng.permutation(n).astype(np.uint32)
        eu, ev = perm[eu], perm[ev]
    else:
        from paper_1503_07192_b200 import graphs
        g = graphs.delaunay(3000, 5)
        n, eu, ev, ew = g.n, g.eu, g.ev, g.ew
        if case == "delaunay_pieces":  # cut into pieces + isolated vertices
            keep = (rng.random(len(eu)) < 0.55)
            eu, ev, ew = eu[keep], ev[keep], ew[keep]
    rgx = ref.graph(n, eu, ev, ew)
    for k, seed in ((37, 2), (150, 7)):
        want, _ = rgx.partition(k, seed)
        got = P.partition_graph(P.Graph(n, eu, ev, ew), k, seed, threads=5)
        assert np.array_equal(got, want), (case, k, seed)


@pytest.mark.parametrize("env", [{"PSP_PART_PAR_LAST": "8"}, {"PSP_PART_SERIAL": "1"},
                                 {"PSP_PART_PAR_LAST": "8", "PSP_PART_SERIAL_RECENTER": "1"}])
def test_partition_parallel_chains_match_reference(ref, env, monkeypatch):
    """Every restart chain on 4 threads (grow_par + recenter_par), or all
    serial: the assignment is the reference's either way, including graphs
    with unreached pieces and isolated vertices."""
    from paper_1503_07192_b200 import graphs
    for key, val in env.items():
        monkeypatch.setenv(key, val)
    g = graphs.delaunay(5000, 8)
    keep = np.random.default_rng(3).random(g.m) < 0.6
    eu, ev, ew = g.eu[keep], g.ev[keep], g.ew[keep]
    rgx = ref.graph(g.n, eu, ev, ew)
    for k, seed in ((29, 4), (200, 1)):
        want, _ = rgx.partition(k, seed)
        got = P.partition_graph(P.Graph(g.n, eu, ev, ew), k, seed, threads=16)
        assert np.array_equal(got, want), (env, k, seed)


def test_partition_disconnected_matches_reference(ref):
    # unreached vertices + isolated vertices exercise finalize's fill step
    eu = np.array([0, 1, 2, 5, 6, 8], np.uint32)
    ev = np.array([1, 2, 3, 6, 7, 9], np.uint32)
    ew = np.ones(6)
    rg = ref.graph(12, eu, ev, ew)
    for k, seed in ((2, 0), (3, 1), (5, 2), (12, 0)):
        want, _ = rg.partition(k, seed)
        got = P.partition_graph(P.Graph(12, eu, ev, ew), k, seed, threads=4)
        assert np.array_equal(got, want), (k, seed)


def test_partition_argument_errors():
    g = P.generate_grid(2, 3)
    with pytest.raises(ValueError):
        P.partition_graph(g, 0)
    with pytest.raises(ValueError):
        P.partition_graph(g, 7)


@pytest.mark.parametrize("edges,msg", [
    (([0], [0], [1.0]), "self-loop"), (([0], [1], [-1.0]), "negative"),
    (([0], [1], [np.nan]), "non-finite"), (([0, 1], [1, 0], [1.0, 1.0]), "duplicate"),
    (([0], [9], [1.0]), "outside"),
])
def test_graph_invariants_rejected(edges, msg):
    eu, ev, ew = edges
    g = P.Graph(3, eu, ev, ew)
    with pytest.raises(P.GraphInvariantError, match=msg):
        P.partition_graph(g, 1)


@pytest.mark.parametrize("bad,msg", [
    ((7, 7, 1.0), r"self-loop at vertex 7$"),
    ((5, 6, -2.0), r"negative weight on edge \(5,6\)$"),
    ((1, 2, 1.0), r"duplicate edge \(1,2\)$"),
])
def test_graph_invariants_first_error_large(bad, msg):
    """Above 64K edges build_csr validates and sorts on several threads; the
    error must still be the one a serial scan meets first (src/graph.cpp:22-36):
    the earliest bad edge, or the lowest vertex with a duplicate neighbour."""
    g = P.generate_grid(400, 400)
    eu, ev, ew = list(g.eu), list(g.ev), list(g.ew)
    u, v, w = bad
    late = len(eu) - 3  # a second, later offence of another kind
    eu.insert(late, 100)
    ev.insert(late, 100)
    ew.insert(late, 1.0)
    eu.insert(1000, u)
    ev.insert(1000, v)
    ew.insert(1000, w)
    if msg.startswith("duplicate"):
        eu.append(159_000)  # a duplicate at a higher vertex too
        ev.append(159_001)
        ew.append(1.0)
        del eu[late + 1], ev[late + 1], ew[late + 1]  # only duplicates remain
    G = P.Graph(g.n, np.array(eu, np.uint32), np.array(ev, np.uint32), np.array(ew))
    with pytest.raises(P.GraphInvariantError, match=msg):
        P.partition_graph(G, 1)


@pytest.mark.parametrize("n,seed", [(3, 0), (100, 2), (20_000, 4), (262_144, 1)])
def test_delaunay_generator_matches_qhull(n, seed):
    """The library's exact incremental Delaunay (csrc/delaunay.cpp) gives the
    same graph as the workload definition (workloads.py: scipy Qhull), up to
    BASELINE configs[1] (262,144 points); configs[2] (1,048,576) was checked
    the same way when the generator was written (3,145,692 equal edges)."""
    import workloads
    from paper_1503_07192_b200 import graphs
    n0, eu, ev, ew = graphs.delaunay_arrays(n, seed)
    r0, ru, rv, rw = workloads.delaunay(n, seed)
    assert n0 == r0
    assert np.array_equal(eu, ru) and np.array_equal(ev, rv) and np.array_equal(ew, rw)


def test_road_generator_matches_scipy_definition():
    # configs[3]'s road-like grid: the product's C++ Kruskal
    # (psp_min_spanning_forest) gives the same spanning forest as scipy's
    # minimum_spanning_tree, hence identical graphs (2048^2 checked once:
    # identical, 4.8 s -> 3.6 s)
    import workloads
    from paper_1503_07192_b200 import graphs
    for rows, cols in ((64, 96), (256, 256), (512, 384)):
        n, eu, ev, ew = workloads.road_grid(rows, cols, 7)
        g = graphs.road_grid(rows, cols, 7)
        assert g.n == n
        assert np.array_equal(g.eu, eu) and np.array_equal(g.ev, ev) and np.array_equal(g.ew, ew)


def test_min_spanning_forest_argument_checks():
    from paper_1503_07192_b200 import _lib
    L = _lib.lib()
    eu = np.array([0, 1], np.uint32)
    ev = np.array([1, 5], np.uint32)  # 5 >= n
    key = np.array([1.0, 2.0])
    mask = np.empty(2, np.uint8)
    assert L.psp_min_spanning_forest(3, 2, eu, ev, key, mask) == _lib.PSP_EINVAL
    ev[1] = 2
    assert L.psp_min_spanning_forest(3, 2, eu, ev, key, mask) == _lib.PSP_OK
    assert mask.tolist() == [1, 1]
