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


def delaunay(n: int, seed: int = 1) -> Graph:
    return _graph(workloads.delaunay(n, seed))


def road_grid(rows: int, cols: int, seed: int = 7, drop: float = 0.10) -> Graph:
    return _graph(workloads.road_grid(rows, cols, seed, drop))


def _grid(rows, cols, weights, seed):
    from . import generate_grid
    g = generate_grid(rows, cols, weights, seed)
    return g.n, g.eu, g.ev, g.ew


def make(name: str) -> tuple[Graph, dict]:
    arrays, cfg = workloads.make_arrays(name, grid=_grid)
    return _graph(arrays), cfg
