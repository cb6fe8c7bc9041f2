"""Synthetic planar inputs for the BASELINE.json configurations as `Graph`s.

The workload definitions live in the repo-root ``workloads.py`` (plain
numpy/scipy, shared with the reference arm of ``bench.py``, which must not
load this package). The grid family is drawn by the library's own
``generate_grid`` (the reference's mt19937_64 generator restated,
csrc/host_graph.cpp).
"""
from __future__ import annotations

import os
import sys

from . import Graph

_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if _ROOT not in sys.path:
    sys.path.insert(0, _ROOT)

import workloads  # noqa: E402

CONFIGS = workloads.CONFIGS


def _graph(arrays) -> Graph:
    n, eu, ev, ew = arrays
    return Graph(n, eu, ev, ew)


def delaunay_arrays(n: int, seed: int = 1):
    """workloads.delaunay with the triangulation by the library's exact
    incremental Delaunay (csrc/delaunay.cpp, ~1.7 s at 1M points instead of
    Qhull's ~12-17 s): same points, same edges, same weights."""
    import ctypes as C

    import numpy as np

    from . import _lib
    rng, pts = workloads.delaunay_points(n, seed)
    cap = 3 * n
    eu = np.empty(cap, np.uint32)
    ev = np.empty(cap, np.uint32)
    m = C.c_uint64()
    _lib.check(_lib.lib().psp_delaunay_edges(n, np.ascontiguousarray(pts, np.float64), cap, eu, ev,
                                              C.byref(m)))
    eu, ev = eu[: m.value].copy(), ev[: m.value].copy()
    return n, eu, ev, workloads.delaunay_weights(rng, m.value)


def delaunay(n: int, seed: int = 1) -> Graph:
    return _graph(delaunay_arrays(n, seed))


def spanning_forest_mask(n, eu, ev, key):
    """C++ Kruskal (psp_min_spanning_forest): the same forest as scipy's for
    distinct keys, without the sparse-matrix round trip."""
    import numpy as np

    from . import _lib
    eu = np.ascontiguousarray(eu, np.uint32)
    ev = np.ascontiguousarray(ev, np.uint32)
    mask = np.empty(len(eu), np.uint8)
    _lib.check(_lib.lib().psp_min_spanning_forest(n, len(eu), eu, ev,
                                                   np.ascontiguousarray(key, np.float64), mask))
    return mask.astype(bool)


def road_grid(rows: int, cols: int, seed: int = 7, drop: float = 0.10) -> Graph:
    return _graph(workloads.road_grid(rows, cols, seed, drop, tree_mask=spanning_forest_mask))


def _grid(rows, cols, weights, seed):
    from . import generate_grid
    g = generate_grid(rows, cols, weights, seed)
    return g.n, g.eu, g.ev, g.ew


def make(name: str) -> tuple[Graph, dict]:
    cfg = dict(CONFIGS[name])
    if cfg["family"] == "delaunay":
        return _graph(delaunay_arrays(cfg["n"], cfg["seed"])), cfg
    arrays, cfg = workloads.make_arrays(name, grid=_grid, tree_mask=spanning_forest_mask)
    return _graph(arrays), cfg
