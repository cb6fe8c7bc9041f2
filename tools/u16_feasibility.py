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


if __name__ == "__main__":
    main()
