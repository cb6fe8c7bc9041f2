"""Preprocessing wall time, repeated: build one configuration several times in
one process (after a small warm-up build, as bench.py does) and print each
build's phases, so the spread between consecutive builds is on record.

  python tools/build_repeat.py --config delaunay1m_k1024 --builds 3
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1503_07192_b200 as P  # noqa: E402
from paper_1503_07192_b200 import graphs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="delaunay1m_k1024")
    ap.add_argument("--builds", type=int, default=3)
    args = ap.parse_args()
    ctx = P.Context(0)
    wg = P.generate_grid(64, 64, (1, 1025), 1)
    P.build_oracle(wg, 16, 1, 0, ctx=ctx).close()
    g, cfg = graphs.make(args.config)
    rows = []
    for i in range(args.builds):
        t0 = time.time()
        o = P.build_oracle(g, cfg["k"], os.cpu_count() or 8, 0, ctx=ctx)
        wall = time.time() - t0
        st = o.stats
        rows.append({"build": i, "wall_s": round(wall, 3),
                     "partition_s": round(st["partition_ms"] / 1e3, 3),
                     "component_apsp_s": round(st["component_apsp_ms"] / 1e3, 3),
                     "boundary_s": round(st["boundary_ms"] / 1e3, 3),
                     "k2_device_s": round(st["k2_device_ms"] / 1e3, 3),
                     "boundary_minus_k2_device_s": round((st["boundary_ms"] - st["k2_device_ms"]) / 1e3, 3),
                     "preprocessing_s": round((st["partition_ms"] + st["component_apsp_ms"]
                                              + st["boundary_ms"]) / 1e3, 3)})
        print(json.dumps(rows[-1]), flush=True)
        o.close()
    pre = [r["preprocessing_s"] for r in rows]
    mean = sum(pre) / len(pre)
    print(json.dumps({"config": args.config, "builds": len(rows), "preprocessing_mean_s": round(mean, 3),
                      "max_dev_pct": round(max(abs(x - mean) for x in pre) / mean * 100, 2)}))


if __name__ == "__main__":
    main()
