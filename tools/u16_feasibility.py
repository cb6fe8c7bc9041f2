"""Feasibility of 16-bit offsets in the query product (VIADDMNMX.U16x2 runs
two relaxations per instruction, profiles/r2/minplus_probe.json: 125.9 vs
62.1 relax/clk/SM; its add wraps at 2^16).

For a query (v1 in C1, v2 in C2) the stitch is min_ij row1[i] + M[i][j] +
col2[j] with M the |B1| x |B2| boundary block. With per-block base min(M) and
per-row base min(row1), the offsets r = row1 - min(row1), m = M - min(M) are
exact in 15 bits when range(row1) + range(M) < 2^15, and then no sum wraps.
This tool measures, on sampled components of a configuration, the spread of
range(M) over blocks and of range(row1) over vertices, and the fraction of
(vertex, block) combinations that fit without any saturation.

  python tools/u16_feasibility.py --config delaunay1m_k1024 --components 24
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1503_07192_b200 as P  # noqa: E402
from paper_1503_07192_b200 import graphs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="delaunay262k_k256")
    ap.add_argument("--components", type=int, default=24)
    args = ap.parse_args()
    g, cfg = graphs.make(args.config)
    o = P.build_oracle(g, cfg["k"], os.cpu_count() or 8, 0)
    scale = 2.0 ** o.stats["fixed_point_shift"]
    bo = o.boundary_offset.astype(np.int64)
    k = o.k
    rng = np.random.default_rng(0)
    comps = rng.choice(k, size=min(args.components, k), replace=False)
    block_ranges, row_ranges = [], []
    fits, total = 0, 0
    for c1 in comps:
        rows = o.boundary_rows(int(c1)) * scale  # |B1| x b, exact integers
        B1 = rows.shape[0]
        ct = o.component_table(int(c1)) * scale  # |C1| x |C1|, boundary-first
        r = ct[:, :B1]  # row1 of every vertex of C1
        rr = np.where(np.isfinite(r), r, np.nan)
        rrange = np.nanmax(rr, axis=1) - np.nanmin(rr, axis=1)
        row_ranges.append(rrange)
        for c2 in range(k):
            blk = rows[:, bo[c2]:bo[c2 + 1]]
            if blk.size == 0:
                continue
            f = blk[np.isfinite(blk)]
            mr = float(f.max() - f.min()) if f.size else 0.0
            block_ranges.append(mr)
            ok = (rrange + mr) < 2 ** 15
            fits += int(ok.sum())
            total += len(rrange)
    br = np.array(block_ranges)
    rr = np.concatenate(row_ranges)
    q = [50, 90, 99, 99.9, 100]
    print(json.dumps({
        "config": args.config, "components_sampled": len(comps), "blocks": len(br),
        "block_range_percentiles": dict(zip(map(str, q), np.percentile(br, q).round(1).tolist())),
        "row1_range_percentiles": dict(zip(map(str, q), np.nanpercentile(rr, q).round(1).tolist())),
        "fraction_vertex_block_fitting_15bit": fits / max(total, 1),
    }))


if __name__ == "__main__" and "--potentials" not in sys.argv:
    main()


def potentials_mode(o, g, scale, comps, queries_per_comp=400, seed=1):
    """Two-sided potentials: M[i][j] = a_i + R[i][j] + b_j with a_i = min_j M,
    b_j = min_i (M - a_i), R >= 0. The 16-bit product runs on R (15-bit
    saturated) with row1 + a and col2 + b folded into the 32-bit ends; a query
    is conclusive when its exact columns beat the lower bound of the
    saturated ones. Returns the conclusive fraction and checks exactness."""
    rng = np.random.default_rng(seed)
    bo = o.boundary_offset.astype(np.int64)
    co = o.component_offset.astype(np.int64)
    assign_orig = o.assignment[o.permutation]
    SAT = 0x7FFF
    tot = conclusive = wrong = 0
    ranges = []
    for c1 in comps:
        rows = o.boundary_rows(int(c1)) * scale
        ct1 = o.component_table(int(c1)) * scale
        B1 = rows.shape[0]
        members = np.flatnonzero(assign_orig == c1)
        for _ in range(queries_per_comp):
            v1 = int(rng.choice(members))
            v2 = int(rng.integers(0, g.n))
            c2 = int(assign_orig[v2])
            l1 = int(o.permutation[v1] - co[c1])
            l2 = int(o.permutation[v2] - co[c2])
            if c2 < c1 or c2 == c1:
                continue  # the kernel orients c1 < c2; same-component adds a cap
            M = rows[:, bo[c2]:bo[c2 + 1]]
            B2 = M.shape[1]
            if B1 == 0 or B2 == 0:
                continue
            ct2 = o.component_table(c2) * scale
            r = ct1[l1, :B1]
            c = ct2[l2, :B2]
            with np.errstate(invalid="ignore"):
                a = np.min(M, axis=1)
                a[~np.isfinite(a)] = 0
                b = np.min(M - a[:, None], axis=0)
                b[~np.isfinite(b)] = 0
                R = M - a[:, None] - b[None, :]
            Rf = np.where(np.isfinite(R), R, np.inf)
            ranges.append(float(np.nanmax(np.where(np.isfinite(Rf), Rf, np.nan))) if np.isfinite(Rf).any() else 0.0)
            rp = r + a
            base_r = np.min(rp[np.isfinite(rp)]) if np.isfinite(rp).any() else 0.0
            r16 = np.minimum(np.where(np.isfinite(rp), rp - base_r, SAT), SAT)
            R16 = np.minimum(np.where(np.isfinite(Rf), Rf, SAT), SAT)
            t16 = np.min(r16[:, None] + R16, axis=0)
            cp = c + b
            exact = t16 < SAT
            cand = np.where(exact, t16 + base_r + cp, np.inf)
            lbv = np.where(~exact, SAT + base_r + cp, np.inf)
            d_exact, lb = float(np.min(cand)), float(np.min(lbv))
            truth = float(np.min(r[:, None] + M + c[None, :]))
            tot += 1
            if d_exact <= lb:
                conclusive += 1
                if d_exact != truth:
                    wrong += 1
    rr = np.array(ranges)
    q = [50, 90, 99, 100]
    return {"queries": tot, "conclusive_fraction": conclusive / max(tot, 1),
            "wrong_when_conclusive": wrong,
            "residual_range_percentiles": dict(zip(map(str, q), np.percentile(rr, q).round(1).tolist()))}


def main2():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="delaunay262k_k256")
    ap.add_argument("--components", type=int, default=8)
    args = ap.parse_args([a for a in sys.argv[1:] if a != "--potentials"])
    g, cfg = graphs.make(args.config)
    o = P.build_oracle(g, cfg["k"], os.cpu_count() or 8, 0)
    scale = 2.0 ** o.stats["fixed_point_shift"]
    comps = np.random.default_rng(0).choice(o.k, size=min(args.components, o.k), replace=False)
    print(json.dumps(dict(potentials_mode(o, g, scale, comps), config=args.config)))


if __name__ == "__main__" and "--potentials" in sys.argv:
    main2()
