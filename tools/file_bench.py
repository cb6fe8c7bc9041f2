"""PSP1 oracle file throughput: build a configuration on
cuda:0, write its oracle file from the device tables (psp_gpu_oracle_save:
f64 conversion + CRC-64/XZ on the GPU, parallel pwrites overlapped with the
next chunk), read it back (psp_gpu_oracle_load: parallel preads streamed to
the device, CRC and conversion there), check
the reloaded oracle answers like the original, report GB/s.

  python tools/file_bench.py --config delaunay262k_k256 [--dir /tmp]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1503_07192_b200 as P  # noqa: E402
from paper_1503_07192_b200 import graphs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="delaunay262k_k256")
    ap.add_argument("--dir", default="/tmp")
    args = ap.parse_args()
    g, cfg = graphs.make(args.config)
    o = P.build_oracle(g, cfg["k"], os.cpu_count() or 8, 0)
    path = os.path.join(args.dir, f"psp_{args.config}.psp1")
    t0 = time.time()
    o.save(path)
    save_s = time.time() - t0
    size = os.path.getsize(path)
    t0 = time.time()
    lo = P.load_oracle(path)
    load_s = time.time() - t0
    v1, v2 = P.random_pairs(g.n, 200_000, 5)
    same = bool(np.array_equal(lo.batch_query(v1, v2), o.batch_query(v1, v2)))
    os.remove(path)
    print(json.dumps({"config": args.config, "file_bytes": size, "save_s": round(save_s, 3),
                      "save_gbs": round(size / save_s / 1e9, 3), "load_s": round(load_s, 3),
                      "load_gbs": round(size / load_s / 1e9, 3), "reloaded_answers_equal": same}))
    assert same


if __name__ == "__main__":
    main()
