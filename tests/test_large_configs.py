"""Full-size parity on the BASELINE configurations (north_star: "bit-exact
(int weights) distances vs the CPU oracle on a 1M-vertex synthetic planar
graph").

Runs by default under ``-m gpu`` on configs[1] (Delaunay 262,144, k=256),
configs[2] (Delaunay 1,048,576, k=1024, the metric's configuration) and
configs[3] (road-like 2048x2048 grid, f32 weights: the tolerance path, with
the component tables dropped during K2 and recomputed); the Delaunay ones
take the benchmarked K2 layout (tile-packed elimination order, asserted via
``k2_positions > b``). ``PSP_LARGE_CONFIGS`` overrides the list, e.g.
``PSP_LARGE_CONFIGS=delaunay262k_k256,delaunay1m_k1024,road4m_k512``.

The check follows the reference's own large-n verification (``cmd_verify``,
proj/tools/psp_main.cpp:237-283): seeded sources, one Dijkstra per source on
the ORIGINAL graph (oracle/psp_oracle.c, f64), GPU distances to sampled
targets compared bit for bit (u32: integer weights) or at relative 1e-5
(f32). Then undirected symmetry through the grouped kernel and agreement of
both query kernels on random batches. A summary line per config goes to
gpurun_out/large_configs.jsonl.
"""
from __future__ import annotations

import json
import os
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import oracle
import paper_1503_07192_b200 as P
from paper_1503_07192_b200 import graphs

pytestmark = pytest.mark.gpu
F32_RTOL = 1e-5
DEFAULT = "delaunay262k_k256,delaunay1m_k1024,road4m_k512"
CONFIGS = [c for c in os.environ.get("PSP_LARGE_CONFIGS", DEFAULT).split(",") if c]
SOURCES = 32
TARGETS = 20_000


@pytest.mark.parametrize("name", CONFIGS)
def test_full_size_config(name, monkeypatch):
    t0 = time.time()
    g, cfg = graphs.make(name)
    gen_s = time.time() - t0
    t0 = time.time()
    o = P.build_oracle(g, cfg["k"], os.cpu_count() or 8, 0)
    build_s = time.time() - t0
    try:
        exact = o.value_kind == P.VALUE_U32
        st = o.stats
        rng = np.random.default_rng(11)
        sources = rng.choice(g.n, size=SOURCES, replace=False)
        targets = rng.choice(g.n, size=TARGETS, replace=False).astype(np.uint32)
        off, to, w = oracle.csr(g.n, g.eu, g.ev, g.ew)
        lib = oracle.Oracle.lib()

        def truth_row(s):
            t = np.empty(g.n)
            lib.pso_dijkstra(g.n, off, to, w, int(s), t)  # ctypes drops the GIL
            return t[targets]

        t0 = time.time()
        with ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 4)) as ex:
            truths = list(ex.map(truth_row, sources))
        dijkstra_s = time.time() - t0
        v1 = np.repeat(sources.astype(np.uint32), TARGETS)
        v2 = np.tile(targets, SOURCES)
        d = o.batch_query(v1, v2)
        t = np.concatenate(truths)
        checked = len(t)
        if exact:
            mismatches = int((d != t).sum())
            max_rel = 0.0
        else:
            rel = np.abs(d - t) / np.maximum(t, 1e-300)
            rel[t == 0] = np.abs(d[t == 0])
            max_rel = float(rel.max())
            mismatches = int((rel > F32_RTOL).sum())
        # the reverse direction of the same pairs (v2 -> v1) also equals Dijkstra
        dr_src = o.batch_query(v2, v1)
        rev_mismatch = int((dr_src != d).sum()) if exact else 0
        # symmetry + kernel agreement on a dense random batch (bitwise for
        # u32; in f32 same-component queries are not turned around, so the
        # two directions may round differently: tolerance, like every f32
        # result)
        a1, a2 = P.random_pairs(g.n, 2_000_000, 3)
        monkeypatch.setenv("PSP_QUERY_KERNEL", "grouped")
        dg = o.batch_query(a1, a2)
        dr = o.batch_query(a2, a1)
        monkeypatch.setenv("PSP_QUERY_KERNEL", "warp")
        dw = o.batch_query(a1[:200_000], a2[:200_000])
        monkeypatch.delenv("PSP_QUERY_KERNEL")
        summary = {"config": name, "n": g.n, "k": cfg["k"], "b": o.b,
                   "value_kind": "u32" if exact else "f32",
                   "graph_gen_s": round(gen_s, 2), "build_s": round(build_s, 2),
                   "k2_device_s": round(st["k2_device_ms"] / 1e3, 3),
                   "k2_positions": st["k2_positions"], "k2_order": st["k2_order"],
                   "k2_spilled": st["k2_spilled"],
                   "sources": SOURCES, "targets": TARGETS,
                   "pairs_checked_vs_dijkstra": checked, "mismatches": mismatches,
                   "reverse_mismatches": rev_mismatch, "dijkstra_s": round(dijkstra_s, 1),
                   "max_rel_err": max_rel, "tolerance": 0.0 if exact else F32_RTOL,
                   "symmetry_max_rel": float(np.max(np.abs(dg - dr) / np.maximum(dg, 1e-300))),
                   "kernels_max_rel": float(np.max(np.abs(dw - dg[:200_000]) /
                                                   np.maximum(dg[:200_000], 1e-300)))}
        os.makedirs("gpurun_out", exist_ok=True)
        with open(os.path.join("gpurun_out", "large_configs.jsonl"), "a") as f:
            f.write(json.dumps(summary) + "\n")
        print(summary)
        assert mismatches == 0, summary
        if o.b >= 128 * 128 and name.startswith("delaunay"):
            # the benchmarked layout: elimination order, tile-packed
            assert st["k2_order"] == 1 and st["k2_positions"] > o.b, summary
        if exact:
            assert rev_mismatch == 0, summary
            assert np.array_equal(dg, dr) and np.array_equal(dw, dg[:200_000])
        else:
            assert np.allclose(dr, dg, rtol=2 * F32_RTOL, atol=0)
            assert np.allclose(dw, dg[:200_000], rtol=2 * F32_RTOL, atol=0)
    finally:
        o.close()
