"""Synthetic planar workloads of BASELINE.json (bench and test tooling).

Plain numpy/scipy: this module imports neither the product package nor the
checkers, so ``bench.py --impl reference`` can build the reference's input
without mapping ``libpsp_gpu.so``. The product's own generators
(``paper_1503_07192_b200.graphs``) must produce identical graphs
(``tests/test_host.py::test_workload_generators_agree``).

The reference only generates (triangulated) grids
(include/psp/generators.hpp:23-30) but loads any edge list
(src/graph_io.cpp:50-91); the Delaunay and road-like families BASELINE.json
names are defined here, seeded and deterministic:

* delaunay(n, seed): Delaunay triangulation (scipy Qhull) of n uniform points
  in [0,1)^2 drawn with numpy default_rng(seed); unique undirected edges in
  lexicographic order; integer weights rng.integers(1, 1025) drawn after the
  points.
* road_grid(rows, cols, seed): "road-like perturbed grid": a 4-neighbour grid
  with ~10% of edges deleted (kept connected via a random spanning tree) and
  jittered coordinates; f32-representable weights = Euclidean length of the
  jittered embedding times U[1,2) rounded to f32 (the tolerance path).

Every generator returns (n, eu, ev, ew): u32, u32, f64 numpy arrays.
"""
from __future__ import annotations

import numpy as np


def delaunay_points(n: int, seed: int = 1):
    rng = np.random.default_rng(seed)
    return rng, rng.random((n, 2))


def unique_edges(tri: np.ndarray, n: int) -> np.ndarray:
    """Unique undirected edges (u < v) of triangles `tri` (t x 3), sorted
    lexicographically, as an (m, 2) int64 array."""
    s = tri.astype(np.int64)
    e = np.concatenate([s[:, [0, 1]], s[:, [1, 2]], s[:, [0, 2]]])
    lo = np.minimum(e[:, 0], e[:, 1])
    hi = np.maximum(e[:, 0], e[:, 1])
    key = np.unique(lo * n + hi)
    return np.stack(np.divmod(key, n), axis=1)


def delaunay_weights(rng, m: int) -> np.ndarray:
    return rng.integers(1, 1025, size=m).astype(np.float64)


def delaunay(n: int, seed: int = 1):
    from scipy.spatial import Delaunay

    rng, pts = delaunay_points(n, seed)
    e = unique_edges(Delaunay(pts).simplices, n)
    w = delaunay_weights(rng, len(e))
    return n, e[:, 0].astype(np.uint32), e[:, 1].astype(np.uint32), w


def scipy_tree_mask(n, eu, ev, key):
    """Edges of the minimum spanning forest under `key` (scipy), as a mask."""
    from scipy.sparse import coo_matrix
    from scipy.sparse.csgraph import minimum_spanning_tree

    mst = minimum_spanning_tree(coo_matrix((key, (eu, ev)), shape=(n, n)).tocsr()).tocoo()
    tree = np.zeros(len(eu), bool)
    # map MST edges back to edge ids (the grid edge (u, v) is unique)
    lin = eu * n + ev
    order = np.argsort(lin)
    mlin = np.minimum(mst.row, mst.col).astype(np.int64) * n + np.maximum(mst.row, mst.col)
    pos = np.searchsorted(lin[order], mlin)
    tree[order[pos]] = True
    return tree


def road_grid(rows: int, cols: int, seed: int = 7, drop: float = 0.10, tree_mask=None):
    """Road-like perturbed grid: jittered 4-neighbour grid, a random spanning
    tree kept (minimum spanning tree under random keys, so deletions never
    disconnect the network) and ~`drop` of the remaining edges removed;
    weights = Euclidean length of the jittered embedding x U[1, 2), rounded to
    f32 (the tolerance path: not dyadic, so the device computes in f32).
    `tree_mask(n, eu, ev, key)` computes the spanning forest (default: scipy;
    the product passes its C++ Kruskal, psp_min_spanning_forest)."""
    tree_mask = tree_mask or scipy_tree_mask
    rng = np.random.default_rng(seed)
    n = rows * cols
    r, c = np.divmod(np.arange(n, dtype=np.int64), cols)
    xy = np.stack([c + rng.uniform(-0.3, 0.3, n), r + rng.uniform(-0.3, 0.3, n)], axis=1)
    right = np.arange(n)[c + 1 < cols]
    down = np.arange(n)[r + 1 < rows]
    eu = np.concatenate([right, down])
    ev = np.concatenate([right + 1, down + cols])
    key = rng.random(len(eu)) + 1.0  # distinct positive keys -> random spanning tree
    tree = tree_mask(n, eu, ev, key)
    keep = tree | (rng.random(len(eu)) >= drop)
    eu, ev = eu[keep], ev[keep]
    length = np.linalg.norm(xy[eu] - xy[ev], axis=1)
    w = (length * rng.uniform(1.0, 2.0, len(eu))).astype(np.float32).astype(np.float64)
    return n, eu.astype(np.uint32), ev.astype(np.uint32), w


CONFIGS = {
    # BASELINE.json configs[0]: runs on the CPU reference too
    "grid64_k16": dict(family="grid", rows=64, cols=64, weights=(1, 1025), seed=1, k=16,
                       queries=10_000),
    # configs[1]
    "delaunay262k_k256": dict(family="delaunay", n=262_144, seed=1, k=256, queries=1_000_000),
    # configs[2]: the metric's configuration ("1M-vertex planar")
    "delaunay1m_k1024": dict(family="delaunay", n=1_048_576, seed=1, k=1024,
                             queries=10_000_000),
    # configs[3]: road-like grid, float32 weights (tolerance path), for
    # preprocessing scaling. k = 512 keeps the u32/f32 tables at ~121 GB per
    # GPU (components 70 GB + boundary graph 51 GB) and minimises FW work.
    "road4m_k512": dict(family="road", rows=2048, cols=2048, seed=7, k=512,
                        queries=10_000_000),
    # mid-size road grid (f32 kernels at a scale that builds in seconds)
    "road1m_k256": dict(family="road", rows=1024, cols=1024, seed=7, k=256, queries=1_000_000),
    # small road grid for tests
    "road64k_k64": dict(family="road", rows=256, cols=256, seed=7, k=64, queries=1_000_000),
}


def make_arrays(name: str, grid=None, tree_mask=None):
    """(n, eu, ev, ew), cfg for a named configuration. The grid family is the
    reference's generate_grid (mt19937_64 weights): pass `grid(rows, cols,
    weights, seed) -> (n, eu, ev, ew)` from whichever library should draw it."""
    cfg = dict(CONFIGS[name])
    fam = cfg["family"]
    if fam == "grid":
        if grid is None:
            raise ValueError("grid family: pass grid=<generator>")
        arrays = grid(cfg["rows"], cfg["cols"], cfg["weights"], cfg["seed"])
    elif fam == "delaunay":
        arrays = delaunay(cfg["n"], cfg["seed"])
    elif fam == "road":
        arrays = road_grid(cfg["rows"], cfg["cols"], cfg["seed"], tree_mask=tree_mask)
    else:
        raise ValueError(fam)
    return arrays, cfg
