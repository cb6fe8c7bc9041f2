"""Full-size parity on the BASELINE configurations (opt-in: minutes per config).

  PSP_LARGE_CONFIGS=delaunay262k_k256,delaunay1m_k1024,road4m_k512 \\
      python -m pytest tests/test_large_configs.py -m gpu -q -s

For each config: build the oracle on cuda:0, then for sampled sources run the
oracle's Dijkstra (oracle/psp_oracle.c, f64, on the ORIGINAL graph) and
compare the GPU distances to random targets: bit-exact for u32 (integer /
dyadic weights), relative error <= 1e-5 for f32 (BASELINE.json north_star).
Also checks undirected symmetry through both query kernels. A summary line
per config is appended to gpurun_out/large_configs.jsonl.
"""
from __future__ import annotations

import json
import os
import time

import numpy as np
import pytest

import oracle
import paper_1503_07192_b200 as P
from paper_1503_07192_b200 import graphs

pytestmark = pytest.mark.gpu
F32_RTOL = 1e-5
CONFIGS = [c for c in os.environ.get("PSP_LARGE_CONFIGS", "").split(",") if c]


@pytest.mark.skipif(not CONFIGS, reason="set PSP_LARGE_CONFIGS to run full-size checks")
@pytest.mark.parametrize("name", CONFIGS or ["none"])
def test_full_size_config(name, monkeypatch):
    g, cfg = graphs.make(name)
    t0 = time.time()
    o = P.build_oracle(g, cfg["k"], os.cpu_count() or 8, 0)
    build_s = time.time() - t0
    exact = o.value_kind == P.VALUE_U32
    rng = np.random.default_rng(11)
    sources = rng.choice(g.n, size=6, replace=False)
    targets = rng.choice(g.n, size=20_000, replace=False)
    max_rel, mismatches, checked = 0.0, 0, 0
    off, to, w = oracle.csr(g.n, g.eu, g.ev, g.ew)
    lib = oracle.Oracle.lib()
    for s in sources:
        truth = np.empty(g.n)
        lib.pso_dijkstra(g.n, off, to, w, int(s), truth)
        v1 = np.full(len(targets), s, np.uint32)
        d = o.batch_query(v1, targets)
        t = truth[targets]
        checked += len(targets)
        if exact:
            mismatches += int((d != t).sum())
        else:
            rel = np.abs(d - t) / np.maximum(t, 1e-300)
            rel[t == 0] = np.abs(d[t == 0])
            max_rel = max(max_rel, float(rel.max()))
            mismatches += int((rel > F32_RTOL).sum())
    # symmetry + kernel agreement on a dense random batch (bitwise for u32;
    # in f32 same-component queries are not turned around, so the two
    # directions may round differently: tolerance, like every f32 result)
    v1, v2 = P.random_pairs(g.n, 2_000_000, 3)
    monkeypatch.setenv("PSP_QUERY_KERNEL", "grouped")
    dg = o.batch_query(v1, v2)
    dr = o.batch_query(v2, v1)
    monkeypatch.setenv("PSP_QUERY_KERNEL", "warp")
    dw = o.batch_query(v1[:200_000], v2[:200_000])
    summary = {"config": name, "n": g.n, "k": cfg["k"], "b": o.b,
               "value_kind": "u32" if exact else "f32", "build_s": round(build_s, 2),
               "k2_device_s": round(o.stats["k2_device_ms"] / 1e3, 3),
               "pairs_checked_vs_dijkstra": checked, "mismatches": mismatches,
               "max_rel_err": max_rel, "tolerance": 0.0 if exact else F32_RTOL,
               "symmetry_max_rel": float(np.max(np.abs(dg - dr) / np.maximum(dg, 1e-300))),
               "kernels_max_rel": float(np.max(np.abs(dw - dg[:200_000]) /
                                               np.maximum(dg[:200_000], 1e-300)))}
    os.makedirs("gpurun_out", exist_ok=True)
    with open(os.path.join("gpurun_out", "large_configs.jsonl"), "a") as f:
        f.write(json.dumps(summary) + "\n")
    print(summary)
    assert mismatches == 0, summary
    if exact:
        assert np.array_equal(dg, dr) and np.array_equal(dw, dg[:200_000])
    else:
        assert np.allclose(dr, dg, rtol=2 * F32_RTOL, atol=0)
        assert np.allclose(dw, dg[:200_000], rtol=2 * F32_RTOL, atol=0)
