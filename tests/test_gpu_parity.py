"""GPU parity: the sm_100a path (through the C-ABI) against the reference.

Checkers: the committed reference fixtures (tests/golden/), the live
reference build (oracle/_ref, travels to the GPU box as a .so) and the C
restatement (oracle/). Integer and dyadic-lattice weights are compared bit
for bit; the f32 path within relative 1e-5 (BASELINE.json north_star).
"""
from __future__ import annotations

import hashlib
import math

import numpy as np
import pytest

import oracle
import paper_1503_07192_b200 as P
from conftest import graph_of

pytestmark = pytest.mark.gpu
INF = math.inf
F32_RTOL = 1e-5  # north_star tolerance for float32 weights

SMALL = ["grid2x3_k2", "grid2x3_k1", "cycle8_k2_s4", "two_squares_k2", "isolated2_k2",
         "grid16_k4", "grid16_k8_lattice", "tri9_k6", "grid10_k2", "tri20_k20_w0",
         "grid32_k32_unit"]


def assert_same_oracle(o: P.GpuOracle, case: dict, full_tables: bool = True):
    k = int(case["k"])
    assert o.k == k and o.n == int(case["n"])
    assert np.array_equal(o.permutation, case["permutation"])
    assert np.array_equal(o.component_offset, case["component_offset"])
    assert np.array_equal(o.boundary_offset, case["boundary_offset"])
    assert np.array_equal(o.boundary_vertex, case["boundary_vertex"])
    assert o.b == int(case["b"])
    assert o.stats["bg_edges"] == int(case["bg_edges"])
    assert o.stats["stored_entries"] == int(case["stored_entries"])
    assert o.stored_entries() == int(case["stored_entries"])
    h = hashlib.sha256()
    for c in range(k):
        ct, bt = o.component_table(c), o.boundary_rows(c)
        if full_tables:
            assert np.array_equal(ct, case[f"ct{c}"]), f"component table {c}"
            assert np.array_equal(bt, case[f"bt{c}"]), f"boundary rows {c}"
        h.update(ct.tobytes())
        h.update(bt.tobytes())
    assert h.digest() == case["tables_sha256"].tobytes()
    d, ops = o.batch_query(case["q_v1"], case["q_v2"], with_ops=True)
    assert np.array_equal(d, case["q_dist"])
    assert np.array_equal(ops, case["q_ops"])


@pytest.mark.parametrize("name", SMALL)
def test_build_oracle_matches_reference_fixture(golden_small, name):
    case = golden_small[name]
    o = P.build_oracle(graph_of(case), int(case["k"]), 1, int(case["seed"]))
    assert o.value_kind == P.VALUE_U32  # integral or dyadic -> exact path
    assert_same_oracle(o, case)
    assert o.stats["peak_table_entries_per_worker"] == int(case["peak_table_entries_per_worker"])


def test_grid2x3_golden_vectors(golden_small):
    # tests/test_oracle.cpp:28-79 and tests/test_query.cpp:30-62
    o = P.build_oracle(P.generate_grid(2, 3), 2, 1, 0)
    path = [0, 2, 1, 2, 0, 1, 1, 1, 0]
    assert o.component_table(0).ravel().tolist() == path
    assert o.component_table(1).ravel().tolist() == path
    assert o.boundary_rows(0).ravel().tolist() == [0, 2, 1, 1, 2, 0, 3, 1]
    assert o.boundary_rows(1).ravel().tolist() == [1, 3, 0, 2, 1, 1, 2, 0]
    assert o.stats["bg_edges"] == 5 and o.stats["stored_entries"] == 34
    assert o.query(0, 5) == (3.0, 6)
    g = P.generate_grid(2, 3)
    truth = oracle.apsp_dense(6, g.eu, g.ev, g.ew)
    v1, v2 = np.divmod(np.arange(36), 6)
    assert np.array_equal(o.batch_query(v1, v2), truth[v1, v2])


def test_same_component_escape_route():
    # tests/test_query.cpp:64-89
    g = P.Graph(8, [0, 1, 2, 3, 4, 5, 6, 0], [1, 2, 3, 4, 5, 6, 7, 7],
                [1, 1, 1, 10, 1, 1, 1, 1])
    o = P.build_oracle(g, 2, 1, 4)
    assert o.query(2, 5)[0] == 5.0
    assert o.query(3, 3)[0] == 0.0


def test_unreachable_and_errors():
    # tests/test_query.cpp:155-172
    o = P.build_oracle(P.Graph(2, [], [], []), 2, 1, 0)
    d, ops = o.query(0, 1)
    assert d == INF and ops == 0
    assert o.query(0, 0)[0] == 0.0
    o2 = P.build_oracle(P.generate_grid(2, 3), 2, 1, 0)
    with pytest.raises(ValueError):
        o2.query(0, 6)
    with pytest.raises(ValueError):
        o2.query(6, 0)
    with pytest.raises(ValueError):
        P.build_oracle(P.generate_grid(2, 3), 7, 1, 0)       # k > n
    with pytest.raises(ValueError):
        P.build_oracle(P.generate_grid(2, 3), 2, 0, 0)       # workers < 1


def test_workers_do_not_change_the_oracle(golden_cfg1):
    # include/psp/oracle.hpp:80-84; tests/test_oracle.cpp:151-160
    g = graph_of(golden_cfg1)
    a = P.build_oracle(g, 16, 1, 0)
    b = P.build_oracle(g, 16, 8, 0)
    for c in range(16):
        assert np.array_equal(a.component_table(c), b.component_table(c))
        assert np.array_equal(a.boundary_rows(c), b.boundary_rows(c))


def test_cfg1_matches_reference(golden_cfg1):
    # BASELINE.json configs[0]: 64x64 grid, integer weights 1..1025, k=16
    case = golden_cfg1
    o = P.build_oracle(graph_of(case), 16, 8, 0)
    assert_same_oracle(o, case, full_tables=False)


def test_cfg1_matches_live_reference_and_restatement(ref):
    rg = ref.generate("grid", 64, 64, (1, 1025), 1)
    ro = rg.build_oracle(16, 8, 0)
    eu, ev, ew = rg.edges()
    g = P.Graph(rg.n, eu, ev, ew)
    o = P.build_oracle(g, 16, 8, 0)
    po = oracle.Oracle(rg.n, eu, ev, ew, 16, ro.permutation, ro.assignment, ro.boundary_flags)
    for c in range(16):
        ct = o.component_table(c)
        assert np.array_equal(ct, ro.component_table(c))
        assert np.array_equal(ct, po.component_table(c))
        bt = o.boundary_rows(c)
        assert np.array_equal(bt, ro.boundary_rows(c))
        assert np.array_equal(bt, po.boundary_rows(c))
    v1, v2 = ref.random_pairs(rg.n, 50_000, 3)
    d, ops = o.batch_query(v1, v2, with_ops=True)
    rd, rops = ro.batch_query(v1, v2, 8, with_ops=True)
    assert np.array_equal(d, rd) and np.array_equal(ops, rops)


@pytest.mark.parametrize("kind,rows,cols,w,gseed", [
    ("grid", 4, 4, None, 0), ("grid", 9, 9, (0.25, 2.0), 5), ("tri", 7, 8, (1.0, 3.0), 1)])
def test_apsp_dense_bitwise(ref, kind, rows, cols, w, gseed):
    # tests/test_shortest_paths.cpp:55-74 (FW == triple loop, any block size)
    rg = ref.generate(kind, rows, cols, w, gseed)
    eu, ev, ew = rg.edges()
    g = P.Graph(rg.n, eu, ev, ew)
    want = rg.apsp_dense(64)
    for bs in (1, 3, 41, 64, 4096):
        assert np.array_equal(P.apsp_dense(g, bs), want)
    d = P.apsp_dense(g)
    assert (np.diag(d) == 0).all() and np.array_equal(d, d.T)
    with pytest.raises(ValueError):
        P.apsp_dense(g, 0)


def test_apsp_dense_disconnected_and_tiles():
    # tests/test_shortest_paths.cpp:59-60 plus sizes straddling the 128 tile
    g = P.Graph(6, [0, 1, 4], [1, 2, 5], [1, 1, 7])
    want = oracle.apsp_dense(6, g.eu, g.ev, g.ew)
    assert np.array_equal(P.apsp_dense(g), want)
    for rows, cols in ((8, 16), (13, 20), (16, 17), (20, 26), (30, 30)):
        gg = P.generate_triangulated_grid(rows, cols, (0.0, 1024.0), rows * cols)
        assert np.array_equal(P.apsp_dense(gg), oracle.apsp_dense(gg.n, gg.eu, gg.ev, gg.ew))


def test_boundary_apsp_clique_omission():
    # tests/test_oracle.cpp:90-112: BG over 3 boundary vertices, clique pair
    # (0,1) omitted because it is unreachable inside its component
    bg = P.Graph(3, [0, 1], [2, 2], [1.0, 1.0])
    t = P.boundary_apsp(bg)
    assert t[:2].ravel().tolist() == [0, 2, 1, 2, 0, 1]
    assert t[2:].ravel().tolist() == [1, 1, 0]


@pytest.mark.parametrize("side,k", [(20, 1), (20, 2), (20, 4), (20, 20), (33, 6), (44, 44)])
def test_exhaustive_all_pairs(side, k):
    # acceptance criterion 1 (acceptance_main.cpp:79-123): all n^2 queries
    g = P.generate_triangulated_grid(side, side, (1.0, 9.0), side)
    truth = oracle.apsp_dense(g.n, g.eu, g.ev, g.ew)
    o = P.build_oracle(g, k, 4, 0)
    v1, v2 = np.divmod(np.arange(g.n * g.n, dtype=np.int64), g.n)
    d = o.batch_query(v1, v2)
    assert np.array_equal(d, truth[v1, v2])


def test_boundary_rows_equal_full_graph_distances():
    # Lemma 1 / acceptance criterion 3 (acceptance_main.cpp:157-180)
    g = P.generate_grid(40, 40, (1, 1025), 8)
    truth = oracle.apsp_dense(g.n, g.eu, g.ev, g.ew)
    o = P.build_oracle(g, 40, 4, 0)
    orig_of_b = o.inverse_permutation[o.boundary_vertex]
    for c in range(o.k):
        rows = o.boundary_rows(c)
        lo = int(o.boundary_offset[c])
        want = truth[np.ix_(orig_of_b[lo: lo + rows.shape[0]], orig_of_b)]
        assert np.array_equal(rows, want)


def test_large_grid_sampled_against_dijkstra():
    # acceptance criterion 2 (acceptance_main.cpp:127-153): 256x256 unit grid,
    # k=128, random queries vs per-source Dijkstra on the original graph
    g = P.generate_grid(256, 256)
    o = P.build_oracle(g, 128, 8, 0)
    v1, v2 = P.random_pairs(g.n, 4000, 17)
    d = o.batch_query(v1, v2)
    order = np.argsort(v1, kind="stable")
    last, truth = -1, None
    for i in order[:1500]:
        if v1[i] != last:
            truth = oracle.dijkstra(g.n, g.eu, g.ev, g.ew, int(v1[i]))
            last = v1[i]
        assert d[i] == truth[v2[i]]
    # undirected symmetry (tests/test_query.cpp:144-153)
    assert np.array_equal(o.batch_query(v2, v1), d)


def test_delaunay_sampled_against_dijkstra():
    from paper_1503_07192_b200 import graphs
    g = graphs.delaunay(20_000, 5)
    o = P.build_oracle(g, 141, 8, 0)
    assert o.value_kind == P.VALUE_U32
    v1, v2 = P.random_pairs(g.n, 20_000, 9)
    d = o.batch_query(v1, v2)
    for s in np.unique(v1)[:25]:
        truth = oracle.dijkstra(g.n, g.eu, g.ev, g.ew, int(s))
        sel = v1 == s
        assert np.array_equal(d[sel], truth[v2[sel]])


def test_f32_tolerance_path():
    # non-dyadic weights -> f32 kernels; relative error <= 1e-5 vs f64
    rng = np.random.default_rng(3)
    g = P.generate_grid(48, 48)
    g = P.Graph(g.n, g.eu, g.ev, rng.uniform(1.0, 2.0, g.m).astype(np.float32).astype(np.float64))
    o = P.build_oracle(g, 24, 4, 0)
    assert o.value_kind == P.VALUE_F32
    truth = oracle.apsp_dense(g.n, g.eu, g.ev, g.ew)
    v1, v2 = np.divmod(np.arange(g.n * g.n, dtype=np.int64)[::7], g.n)
    d = o.batch_query(v1, v2)
    t = truth[v1, v2]
    rel = np.abs(d - t) / np.maximum(t, 1e-300)
    rel[t == 0] = np.abs(d[t == 0])
    assert rel.max() <= F32_RTOL, rel.max()
    # forcing u32 on non-dyadic weights is refused, not silently rounded
    with pytest.raises(ValueError):
        P.build_oracle(g, 24, 1, 0, value_kind=P.VALUE_U32)


def test_disconnected_components_give_empty_boundary_graph(golden_small):
    # tests/test_oracle.cpp:114-122
    case = golden_small["two_squares_k2"]
    o = P.build_oracle(graph_of(case), 2, 1, 0)
    assert o.b == 0 and o.stats["bg_edges"] == 0 and o.stored_entries() == 32


def test_minplus_peak_probe(ctx):
    r_u32, mhz = ctx.minplus_peak(P.VALUE_U32)
    r_f32, _ = ctx.minplus_peak(P.VALUE_F32)
    assert r_u32 > 1e12 and r_f32 > 1e12 and mhz > 500


@pytest.mark.parametrize("kernel", ["warp", "grouped", "cta"])
def test_both_query_kernels_bitwise(monkeypatch, golden_cfg1, kernel):
    # the dense (grouped by component pair) and sparse (warp per query)
    # kernels must return the reference's distances bit for bit
    monkeypatch.setenv("PSP_QUERY_KERNEL", kernel)
    case = golden_cfg1
    o = P.build_oracle(graph_of(case), 16, 8, 0)
    d, ops = o.batch_query(case["q_v1"], case["q_v2"], with_ops=True)
    assert np.array_equal(d, case["q_dist"]) and np.array_equal(ops, case["q_ops"])
    g = P.generate_triangulated_grid(33, 33, (1.0, 9.0), 4)
    truth = oracle.apsp_dense(g.n, g.eu, g.ev, g.ew)
    o2 = P.build_oracle(g, 11, 4, 0)
    v1, v2 = np.divmod(np.arange(g.n * g.n, dtype=np.int64)[::3], g.n)
    assert np.array_equal(o2.batch_query(v1, v2), truth[v1, v2])
    # f32 tolerance path through the same kernel
    rng = np.random.default_rng(5)
    gf = P.Graph(g.n, g.eu, g.ev, rng.uniform(1.0, 2.0, g.m).astype(np.float32).astype(np.float64))
    tf = oracle.apsp_dense(gf.n, gf.eu, gf.ev, gf.ew)
    of = P.build_oracle(gf, 11, 4, 0)
    assert of.value_kind == P.VALUE_F32
    df = of.batch_query(v1, v2)
    t = tf[v1, v2]
    assert (np.abs(df - t) <= F32_RTOL * np.maximum(t, 1e-300)).all()


def test_large_boundaries_query_paths(monkeypatch):
    # few components -> boundaries far above one 64-column pass / 32-row
    # chunk / 512-column warp window; exercises every loop boundary
    g = P.generate_grid(90, 90, (1, 1025), 6)
    o = P.build_oracle(g, 3, 8, 0)
    assert max(np.diff(o.boundary_offset)) > 64
    v1, v2 = P.random_pairs(g.n, 3000, 8)
    want = np.array([oracle.dijkstra(g.n, g.eu, g.ev, g.ew, int(s))[int(t)]
                     for s, t in zip(v1[:200], v2[:200])])
    dw = None
    for kernel in ("warp", "grouped", "cta"):
        monkeypatch.setenv("PSP_QUERY_KERNEL", kernel)
        d = o.batch_query(v1, v2)
        assert np.array_equal(d[:200], want)
        if dw is None:
            dw = d
        else:
            assert np.array_equal(d, dw)


@pytest.mark.parametrize("spill", [False, True])
def test_multigpu_sharded_build(spill):
    # BG Floyd-Warshall row-sharded over every visible GPU (NCCL), checked
    # bitwise against the reference fixture and a single-GPU build; `spill`
    # forces the path where the component tables are dropped during K2 and
    # recomputed (component-sharded K1 + NVLink broadcast) afterwards
    import subprocess
    import sys
    n = P._lib.lib().psp_gpu_device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--standalone",
                        "--nproc-per-node", str(min(n, 4)), os.path.join(root, "tools", "mgpu_check.py")],
                       capture_output=True, text=True, timeout=900,
                       env=dict(os.environ, **({"PSP_K2_FORCE_SPILL": "1"} if spill else {})))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count("bit-exact") == min(n, 4)


@pytest.mark.parametrize("name", ["grid2x3_k2", "cycle8_k2_s4", "grid16_k8_lattice", "tri20_k20_w0",
                                  "isolated2_k2", "two_squares_k2"])
def test_import_oracle_from_reference_tables(golden_small, name):
    # psp_gpu_oracle_import: device oracle from host (reference-built) tables
    case = golden_small[name]
    n, k = int(case["n"]), int(case["k"])
    perm = case["permutation"]
    assign_r = np.empty(n, np.uint32)
    assign_r[perm] = case["assignment"]
    o = P.import_oracle(n, k, perm, assign_r, case["component_offset"], case["boundary_offset"],
                        [case[f"ct{c}"] for c in range(k)], [case[f"bt{c}"] for c in range(k)])
    assert o.value_kind == P.VALUE_U32
    for c in range(k):
        assert np.array_equal(o.component_table(c), case[f"ct{c}"])
        assert np.array_equal(o.boundary_rows(c), case[f"bt{c}"])
    d, ops = o.batch_query(case["q_v1"], case["q_v2"], with_ops=True)
    assert np.array_equal(d, case["q_dist"]) and np.array_equal(ops, case["q_ops"])


def test_edge_shapes():
    # a single vertex, k = 1
    o = P.build_oracle(P.Graph(1, [], [], []), 1, 1, 0)
    assert o.query(0, 0) == (0.0, 0) and o.b == 0
    # k = n: every vertex its own component (tests/test_partition.cpp:94-99)
    g = P.generate_grid(4, 5, (1, 9), 2)
    o = P.build_oracle(g, g.n, 2, 0)
    truth = oracle.apsp_dense(g.n, g.eu, g.ev, g.ew)
    v1, v2 = np.divmod(np.arange(g.n * g.n), g.n)
    assert np.array_equal(o.batch_query(v1, v2), truth[v1, v2])
    # caller-supplied partition with an empty component (make_partition
    # allows it): component 1 owns nothing
    g = P.generate_grid(6, 6, (1, 9), 5)
    assign = np.where(np.arange(g.n) % 6 < 3, 0, 2).astype(np.uint32)
    o = P.build_partitioned(g, 3, assign)
    assert o.component_size(1) == 0
    truth = oracle.apsp_dense(g.n, g.eu, g.ev, g.ew)
    v1, v2 = np.divmod(np.arange(g.n * g.n), g.n)
    for kernel in ("grouped", "warp"):
        import os
        os.environ["PSP_QUERY_KERNEL"] = kernel
        try:
            assert np.array_equal(o.batch_query(v1, v2), truth[v1, v2])
        finally:
            os.environ.pop("PSP_QUERY_KERNEL")
    # empty batch
    assert o.batch_query([], []).shape == (0,)


@pytest.mark.gpu
def test_block_query_layout_matches_tile_arena(monkeypatch, golden_cfg1):
    """The block query layout (default) and the tile-arena fallback give the
    same distances, and both match the reference fixture."""
    from paper_1503_07192_b200 import graphs
    z = golden_cfg1
    cases = [(P.Graph(int(z["n"]), z["eu"], z["ev"], z["ew"]), 16), (graphs.delaunay(20_000, 4), 97)]
    for g, k in cases:
        monkeypatch.setenv("PSP_QUERY_LAYOUT", "tiles")
        ot = P.build_oracle(g, k, 4, 0)
        monkeypatch.delenv("PSP_QUERY_LAYOUT")
        ob = P.build_oracle(g, k, 4, 0)
        v1, v2 = P.random_pairs(g.n, 300_000, 7)
        assert np.array_equal(ob.batch_query(v1, v2), ot.batch_query(v1, v2))
    assert np.array_equal(ob.batch_query(v1[:10], v2[:10]), ot.batch_query(v1[:10], v2[:10]))
    o = P.build_oracle(cases[0][0], 16, 4, 0)
    assert np.array_equal(o.batch_query(z["q_v1"], z["q_v2"]), z["q_dist"])


@pytest.mark.gpu
def test_query_pipe_matches_batch_query(golden_cfg1):
    """psp_gpu_query_pipe_*: pipelined host batches give batch_query's answers;
    a bad id fails wait() and the pipe stays usable."""
    z = golden_cfg1
    o = P.build_oracle(graph_of(z), 16, 4, 0)
    for depth in (1, 2, 3):
        pipe = o.query_pipe(depth)
        sizes = [1, 10_000, 77, 250_000, 3, 100_000, 5_000]
        batches = []
        for i, m in enumerate(sizes):
            v1, v2 = P.random_pairs(o.n, m, 100 + i)
            out = np.empty(m, np.float64)
            pipe.submit(v1, v2, out)
            batches.append((v1, v2, out))
        pipe.wait()
        for v1, v2, out in batches:
            assert np.array_equal(out, o.batch_query(v1, v2))
        fixture = np.empty(len(z["q_v1"]), np.float64)
        pipe.submit(z["q_v1"], z["q_v2"], fixture)
        pipe.wait()
        assert np.array_equal(fixture, z["q_dist"])
        bad1 = np.array([0, o.n], np.uint32)
        pipe.submit(z["q_v1"][:2], z["q_v2"][:2], np.empty(2))
        pipe.submit(bad1, bad1[::-1].copy(), np.empty(2))
        with pytest.raises(ValueError):
            pipe.wait()
        again = np.empty(len(z["q_v1"]), np.float64)
        pipe.submit(z["q_v1"], z["q_v2"], again)
        pipe.wait()
        assert np.array_equal(again, z["q_dist"])
        pipe.close()


@pytest.mark.gpu
def test_k2_order_and_sparse_walk_do_not_change_the_tables(monkeypatch, golden_cfg1):
    """The K2 elimination order (bg_order.hpp, permuted back to reference
    ids) and the sparse phase-3 walk give the same boundary tables and
    answers as the dense FW in the reference numbering."""
    from paper_1503_07192_b200 import graphs
    z = golden_cfg1
    cases = [(graph_of(z), 16), (graphs.delaunay(20_000, 4), 97),
             (P.generate_grid(40, 60, (1, 9), 3), 24)]
    for g, k in cases:
        monkeypatch.setenv("PSP_FW_DENSE", "1")
        monkeypatch.setenv("PSP_BG_ORDER", "natural")
        od = P.build_oracle(g, k, 4, 0)
        monkeypatch.delenv("PSP_FW_DENSE")
        on = P.build_oracle(g, k, 4, 0)  # sparse walk, reference numbering
        monkeypatch.setenv("PSP_BG_ORDER", "component")
        oc = P.build_oracle(g, k, 4, 0)  # sparse walk, component order
        monkeypatch.delenv("PSP_BG_ORDER")
        oo = P.build_oracle(g, k, 4, 0)  # sparse walk, piece order (default)
        for c in range(k):
            ref = od.boundary_rows(c)
            assert np.array_equal(on.boundary_rows(c), ref)
            assert np.array_equal(oc.boundary_rows(c), ref)
            assert np.array_equal(oo.boundary_rows(c), ref)
        assert oo.stats["k2_relaxations"] <= od.stats["k2_relaxations"]
        v1, v2 = P.random_pairs(g.n, 200_000, 9)
        d = od.batch_query(v1, v2)
        for o in (on, oc, oo):
            assert np.array_equal(o.batch_query(v1, v2), d)


@pytest.mark.gpu
def test_k2_tile_packed_layout_matches_dense_walk(monkeypatch, golden_cfg1):
    """The tile-packed K2 layout (bg_pack: units swapped to avoid straddling
    a tile, padding positions = isolated vertices) is what cfg2-cfg4 run;
    it switches on by itself only from 128 tiles per side. PSP_BG_PACK=force
    puts small graphs on it, and the tables and answers must equal the dense
    walk in reference numbering bit for bit."""
    from paper_1503_07192_b200 import graphs
    z = golden_cfg1
    cases = [(graph_of(z), 16), (graphs.delaunay(20_000, 4), 97),
             (graphs.delaunay(60_000, 5), 160), (P.generate_grid(90, 90, (0.25, 2.0), 4), 48)]
    for g, k in cases:
        monkeypatch.setenv("PSP_FW_DENSE", "1")
        monkeypatch.setenv("PSP_BG_ORDER", "natural")
        od = P.build_oracle(g, k, 4, 0)
        monkeypatch.delenv("PSP_FW_DENSE")
        monkeypatch.delenv("PSP_BG_ORDER")
        monkeypatch.setenv("PSP_BG_PACK", "force")
        op = P.build_oracle(g, k, 4, 0)
        monkeypatch.delenv("PSP_BG_PACK")
        assert op.stats["k2_order"] == 1
        # padding positions exist, so the packing really ran
        assert op.stats["k2_positions"] > op.b, (op.stats["k2_positions"], op.b)
        for c in range(k):
            assert np.array_equal(op.boundary_rows(c), od.boundary_rows(c))
            assert np.array_equal(op.component_table(c), od.component_table(c))
        v1, v2 = P.random_pairs(g.n, 300_000, 13)
        assert np.array_equal(op.batch_query(v1, v2), od.batch_query(v1, v2))


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["recompute", "host"])
def test_k2_spill_paths_give_the_same_oracle(monkeypatch, golden_cfg1, mode):
    """When the ordered K2 table does not fit beside the component tables
    (cfg4), the component tables leave the device for the boundary-graph FW:
    dropped and recomputed (default) or parked in host memory
    (PSP_K2_SPILL=host). Forced here on small graphs, both must give the
    same component tables, boundary tables and answers."""
    from paper_1503_07192_b200 import graphs
    z = golden_cfg1
    cases = [(graph_of(z), 16), (graphs.delaunay(20_000, 4), 97)]
    for g, k in cases:
        base = P.build_oracle(g, k, 4, 0)
        monkeypatch.setenv("PSP_K2_FORCE_SPILL", "1")
        if mode == "host":
            monkeypatch.setenv("PSP_K2_SPILL", "host")
        o = P.build_oracle(g, k, 4, 0)
        monkeypatch.delenv("PSP_K2_FORCE_SPILL")
        monkeypatch.delenv("PSP_K2_SPILL", raising=False)
        for c in range(k):
            assert np.array_equal(o.component_table(c), base.component_table(c))
            assert np.array_equal(o.boundary_rows(c), base.boundary_rows(c))
        v1, v2 = P.random_pairs(g.n, 100_000, 5)
        assert np.array_equal(o.batch_query(v1, v2), base.batch_query(v1, v2))


@pytest.mark.gpu
def test_concurrent_device_queries_on_own_streams(golden_cfg1):
    """psp_gpu_query_batch_device from 4 host threads at once, each on its
    own CUDA stream with its own pairs (the reference promises concurrent
    queries are safe, proj/README.md:122-126): every batch equals the
    serial answer bit for bit."""
    import threading

    import torch
    from paper_1503_07192_b200 import graphs
    g = graphs.delaunay(20_000, 4)
    o = P.build_oracle(g, 97, 4, 0)
    dev = torch.device("cuda", 0)
    nthreads, iters, batch = 4, 12, 50_000
    v1, v2 = P.random_pairs(g.n, nthreads * iters * batch, 21)
    want = o.batch_query(v1, v2)
    d1 = torch.from_numpy(v1.view(np.int32)).to(dev)
    d2 = torch.from_numpy(v2.view(np.int32)).to(dev)
    out = torch.empty(len(v1), dtype=torch.float64, device=dev)
    torch.cuda.synchronize()
    errors = []

    def worker(t):
        try:
            st = torch.cuda.Stream(device=dev)
            for i in range(iters):
                j = (t * iters + i) * batch
                # vary the size so workspaces grow while other threads run
                cnt = batch - (i % 3) * 1000
                o.batch_query_device(d1[j:].data_ptr(), d2[j:].data_ptr(), out[j:].data_ptr(),
                                     cnt, st.cuda_stream)
                if i % 3:
                    o.batch_query_device(d1[j + cnt:].data_ptr(), d2[j + cnt:].data_ptr(),
                                         out[j + cnt:].data_ptr(), batch - cnt, st.cuda_stream)
            st.synchronize()
        except Exception as e:  # noqa: BLE001
            errors.append(e)

    th = [threading.Thread(target=worker, args=(t,)) for t in range(nthreads)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    torch.cuda.synchronize()
    assert not errors, errors
    assert np.array_equal(out.cpu().numpy(), want)


@pytest.mark.gpu
def test_point_query_server(monkeypatch):
    """Host calls with <= 32 pairs (the reference's query(o, u, v) in a loop)
    go to the resident point-query server CTA (query_server): answers equal
    the reference's (all-pairs Floyd-Warshall) bit for bit, across server
    idle-outs and relaunches, for every request size 1..32, with the
    reference's error on an out-of-range id."""
    import time
    g = P.generate_triangulated_grid(33, 33, (1.0, 9.0), 4)
    truth = oracle.apsp_dense(g.n, g.eu, g.ev, g.ew)
    o = P.build_oracle(g, 11, 4, 0)
    rng = np.random.default_rng(3)
    v1 = rng.integers(0, g.n, 4000)
    v2 = rng.integers(0, g.n, 4000)
    t0 = time.perf_counter()
    for i in range(2000):
        d, ops = o.query(int(v1[i]), int(v2[i]))
        assert d == truth[v1[i], v2[i]]
    per_query_us = (time.perf_counter() - t0) / 2000 * 1e6
    print(f"point query: {per_query_us:.2f} us per call through the Python binding")
    # the server idles out (200 us default) between these: relaunch path
    for i in range(2000, 2040):
        time.sleep(0.001)
        assert o.query(int(v1[i]), int(v2[i]))[0] == truth[v1[i], v2[i]]
    # every request size of the mailbox
    pos = 0
    for cnt in range(1, 33):
        a, b = v1[pos:pos + cnt], v2[pos:pos + cnt]
        assert np.array_equal(o.batch_query(a, b), truth[a, b])
        pos += cnt
    # a 1 us idle time makes the exit race the next request constantly
    monkeypatch.setenv("PSP_SERVER_IDLE_US", "1")
    for i in range(2040, 3000):
        assert o.query(int(v1[i]), int(v2[i]))[0] == truth[v1[i], v2[i]]
    monkeypatch.delenv("PSP_SERVER_IDLE_US")
    with pytest.raises(ValueError):
        o.query(0, g.n)
    assert o.query(1, 2)[0] == truth[1, 2]  # still serving after the error
    # f32 tables through the same server
    gf = P.Graph(g.n, g.eu, g.ev, rng.uniform(1.0, 2.0, g.m).astype(np.float32).astype(np.float64))
    tf = oracle.apsp_dense(gf.n, gf.eu, gf.ev, gf.ew)
    of = P.build_oracle(gf, 11, 4, 0)
    for i in range(300):
        d = of.query(int(v1[i]), int(v2[i]))[0]
        t = tf[v1[i], v2[i]]
        assert abs(d - t) <= F32_RTOL * max(t, 1e-300)
    # the server and the batch kernels agree on f32 rounding exactly
    monkeypatch.setenv("PSP_QUERY_KERNEL", "grouped")
    db = of.batch_query(v1[:300], v2[:300])
    ds = np.array([of.query(int(v1[i]), int(v2[i]))[0] for i in range(300)])
    assert np.array_equal(db, ds)


@pytest.mark.gpu
def test_sparse_grouping_matches_dense(monkeypatch):
    """Batches far smaller than k^2 are grouped by a radix sort of their pair
    keys (runs as bins) instead of the k^2-bin counting sort: every size,
    including runs of a single query and the tiny-batch query_cta path,
    answers bit for bit like the dense grouping and the Dijkstra truth."""
    from paper_1503_07192_b200 import graphs
    g = graphs.delaunay(20_000, 4)
    o = P.build_oracle(g, 97, 4, 0)  # k^2 = 9409 (sparse forced by PSP_GROUPING)
    v1, v2 = P.random_pairs(g.n, 6000, 31)
    truth = np.array([oracle.dijkstra(g.n, g.eu, g.ev, g.ew, int(s))[int(t)]
                      for s, t in zip(v1[:40], v2[:40])])
    for cnt in (1, 7, 512, 513, 1500, 2352, 2353, 6000):
        a, b = v1[:cnt], v2[:cnt]
        d_auto = o.batch_query(a, b)
        monkeypatch.setenv("PSP_QUERY_KERNEL", "grouped")
        monkeypatch.setenv("PSP_GROUPING", "dense")
        d_dense = o.batch_query(a, b)
        monkeypatch.setenv("PSP_GROUPING", "sparse")
        d_sparse = o.batch_query(a, b)
        monkeypatch.delenv("PSP_GROUPING")
        monkeypatch.delenv("PSP_QUERY_KERNEL")
        assert np.array_equal(d_auto, d_dense), cnt
        assert np.array_equal(d_sparse, d_dense), cnt
        m = min(cnt, 40)
        assert np.array_equal(d_auto[:m], truth[:m]), cnt


@pytest.mark.gpu
@pytest.mark.parametrize("sat", [None, "0x3F", "0x400"])
def test_u16_residual_product_matches_u32(monkeypatch, golden_cfg1, sat):
    """The 16-bit residual product (two-sided block potentials, 15-bit
    saturated offsets, VIADDMNMX.U16x2; opt-in via PSP_QUERY_U16=1) answers
    every dense batch bit for bit like the u32 product. A tiny saturation (PSP_U16_SAT, tests only)
    sends most queries through the lower-bound test and the u32 fallback,
    which must not change a single answer either."""
    from paper_1503_07192_b200 import graphs
    z = golden_cfg1
    cases = [(graph_of(z), 16, 200_000), (graphs.delaunay(20_000, 4), 97, 400_000),
             (P.generate_grid(90, 90, (0.25, 2.0), 4), 48, 300_000),
             (P.Graph(8, [0, 1, 2, 4, 5], [1, 2, 3, 5, 6], [1, 1, 1, 2, 2]), 2, 5_000)]
    for g, k, cnt in cases:
        monkeypatch.delenv("PSP_QUERY_U16", raising=False)
        o32 = P.build_oracle(g, k, 4, 0)
        monkeypatch.setenv("PSP_QUERY_U16", "1")  # opt-in path (slower on cfg3)
        if sat:
            monkeypatch.setenv("PSP_U16_SAT", sat)
        o16 = P.build_oracle(g, k, 4, 0)
        monkeypatch.delenv("PSP_U16_SAT", raising=False)
        if o16.b:  # the 16-bit layout exists wherever there is a boundary table
            assert o16.stats["device_bytes"] > o32.stats["device_bytes"]
        v1, v2 = P.random_pairs(g.n, cnt, 41)
        monkeypatch.setenv("PSP_QUERY_KERNEL", "grouped")
        d16 = o16.batch_query(v1, v2)
        monkeypatch.delenv("PSP_QUERY_U16")
        d32 = o32.batch_query(v1, v2)
        monkeypatch.delenv("PSP_QUERY_KERNEL")
        assert np.array_equal(d16, d32), (k, sat, int((d16 != d32).sum()))
        truth = np.array([oracle.dijkstra(g.n, g.eu, g.ev, g.ew, int(s))[int(t)]
                          for s, t in zip(v1[:30], v2[:30])])
        assert np.array_equal(d16[:30], truth)
