"""Regenerate tests/golden/*.npz from the UNMODIFIED reference build.

Run in the dev container (needs oracle/_ref/libpspref.so, built from
/root/reference/proj/src by oracle/Makefile):

    python tests/golden/make_golden.py

Every fixture stores the graph (edge list), the partition the reference
chose (assignment in original ids, permutation, offsets), its BuildStats
counters, its tables (small cases: complete f64 tables; cfg1: SHA-256 of the
concatenated f64 tables) and seeded query answers (distance + minplus_ops).
"""
from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402


def cycle8_heavy():
    # tests/test_query.cpp:21-27: 8-cycle, unit weights, edge 3-4 costs 10
    eu = [0, 1, 2, 3, 4, 5, 6, 0]
    ev = [1, 2, 3, 4, 5, 6, 7, 7]
    ew = [1, 1, 1, 10, 1, 1, 1, 1]
    return 8, eu, ev, ew


def two_squares():
    # tests/test_oracle.cpp:114-122
    eu = [0, 1, 2, 0, 4, 5, 6, 4]
    ev = [1, 2, 3, 3, 5, 6, 7, 7]
    return 8, eu, ev, [1.0] * 8


SMALL = [
    # name, graph source, k, seed
    ("grid2x3_k2", ("grid", 2, 3, None, 0), 2, 0),           # tests/test_oracle.cpp:28-79
    ("grid2x3_k1", ("grid", 2, 3, None, 0), 1, 0),           # tests/test_oracle.cpp:81-88
    ("cycle8_k2_s4", ("edges", cycle8_heavy), 2, 4),         # tests/test_query.cpp:64-89
    ("two_squares_k2", ("edges", two_squares), 2, 0),        # tests/test_oracle.cpp:114-122
    ("isolated2_k2", ("edges", lambda: (2, [], [], [])), 2, 0),  # tests/test_query.cpp:155-164
    ("grid16_k4", ("grid", 16, 16, None, 0), 4, 0),          # tests/test_query.cpp:91-106
    ("grid16_k8_lattice", ("grid", 16, 16, (0.5, 2.0), 9), 8, 0),  # tests/test_query.cpp:125-142
    ("tri9_k6", ("tri", 9, 9, (1.0, 3.0), 4), 6, 0),         # tests/test_query.cpp:144-153
    ("grid10_k2", ("grid", 10, 10, None, 0), 2, 0),          # tests/test_oracle.cpp:124-149
    ("tri20_k20_w0", ("tri", 20, 20, (0.0, 1024.0), 3), 20, 0),
    ("grid32_k32_unit", ("grid", 32, 32, None, 0), 32, 0),   # acceptance crit 4 shape
]


def graph_of(R, src):
    if src[0] in ("grid", "tri"):
        _, r, c, w, s = src
        return R.generate(src[0], r, c, w, s)
    n, eu, ev, ew = src[1]()
    return R.graph(n, np.array(eu, np.uint32), np.array(ev, np.uint32), np.array(ew, np.float64))


def capture(R, rg, k, seed, nq, qseed, full_tables: bool):
    o = rg.build_oracle(k, 1, seed)
    eu, ev, ew = rg.edges()
    v1, v2 = R.random_pairs(rg.n, nq, qseed)
    dist, ops = o.batch_query(v1, v2, 1, with_ops=True)
    inv = np.empty(rg.n, np.int64)
    inv[o.permutation] = np.arange(rg.n)
    assignment = o.assignment[o.permutation]  # reordered -> original id space
    out = dict(n=rg.n, k=k, seed=seed, eu=eu, ev=ev, ew=ew, assignment=assignment,
               permutation=o.permutation, component_offset=o.component_offset,
               boundary_offset=o.boundary_offset, boundary_vertex=o.boundary_vertex,
               b=o.b, bg_edges=int(o.stats["bg_edges"]),
               stored_entries=int(o.stats["stored_entries"]),
               peak_table_entries_per_worker=int(o.stats["peak_table_entries_per_worker"]),
               q_v1=v1, q_v2=v2, q_dist=dist, q_ops=ops)
    h = hashlib.sha256()
    for c in range(k):
        ct = o.component_table(c)
        br = o.boundary_rows(c)
        h.update(ct.tobytes())
        h.update(br.tobytes())
        if full_tables:
            out[f"ct{c}"] = ct
            out[f"bt{c}"] = br
    out["tables_sha256"] = np.frombuffer(h.digest(), np.uint8)
    return out


def main():
    R = oracle.RefLib()
    small = {}
    for name, src, k, seed in SMALL:
        rg = graph_of(R, src)
        small[name] = capture(R, rg, k, seed, 300, 7, full_tables=True)
        print(name, "n", rg.n, "b", small[name]["b"], "bg_edges", small[name]["bg_edges"])
    flat = {f"{name}/{key}": val for name, d in small.items() for key, val in d.items()}
    np.savez_compressed(os.path.join(HERE, "ref_small.npz"), **flat)

    # BASELINE configs[0]: 64x64 grid, uniform(1,1025) seed 1, k=16, 10k queries
    rg = R.generate("grid", 64, 64, (1, 1025), 1)
    cfg1 = capture(R, rg, 16, 0, 10_000, 42, full_tables=False)
    np.savez_compressed(os.path.join(HERE, "ref_cfg1.npz"), **cfg1)
    print("cfg1 b", cfg1["b"], "bg_edges", cfg1["bg_edges"], "stored", cfg1["stored_entries"])

    # random_pairs stream pin: first pairs of ref::random_pairs
    v1, v2 = R.random_pairs(1000, 16, 123)
    np.savez(os.path.join(HERE, "random_pairs_n1000_s123.npz"), v1=v1, v2=v2)


def cluster_fixture(R=None):
    """ClusterSim::run_batch (src/cluster.cpp:225-231) on BASELINE configs[0]
    with p = 2 and 4 workers, both placement policies: distances and ledger
    rows, for the multi-GPU routed-query check (tools/routed_check.py)."""
    R = R or oracle.RefLib()
    rg = R.generate("grid", 64, 64, (1, 1025), 1)
    ro = rg.build_oracle(16, 4, 0)
    z = np.load(os.path.join(HERE, "ref_cfg1.npz"))
    v1, v2 = z["q_v1"][:4000], z["q_v2"][:4000]
    out = {"v1": v1, "v2": v2}
    for p in (2, 4):
        for pol in (0, 1):
            dist, rec = ro.cluster_run_batch(p, v1, v2, pol)
            out[f"p{p}_pol{pol}_dist"] = dist
            out[f"p{p}_pol{pol}_ledger"] = rec
            print(f"cluster p={p} policy={pol}: {len(rec)} transfers, {int(rec[:, 4].sum())} bytes")
    np.savez_compressed(os.path.join(HERE, "ref_cluster_cfg1.npz"), **out)


if __name__ == "__main__":
    import sys
    if sys.argv[1:] == ["cluster"]:
        cluster_fixture()
    else:
        main()
        cluster_fixture()
