"""Graph ingestion throughput: psp::load_graph (reference build, one host
thread, getline + from_chars, DIMACS via std::map) against load_graph here
(file -> pinned -> HBM, parsed on the GPU). Both read the same file, written
by save_graph; the graphs are checked equal. One JSON line per format.

  python tools/ingest_bench.py [--config road4m_k512] [--reps 3]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1503_07192_b200 as P  # noqa: E402
from paper_1503_07192_b200 import graphs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="road4m_k512")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--no-reference", action="store_true")
    args = ap.parse_args()
    g, _ = graphs.make(args.config)
    ctx = P.Context(0)
    ref = None
    if not args.no_reference:
        try:
            import oracle
            ref = oracle.RefLib()
        except Exception as e:  # noqa: BLE001
            print(f"reference unavailable: {e}", file=sys.stderr)
    with tempfile.TemporaryDirectory() as tmp:
        for fmt in (P.EDGE_LIST, P.DIMACS):
            path = os.path.join(tmp, f"g.{fmt}")
            t = time.perf_counter()
            P.save_graph(g, path, fmt)
            save_s = time.perf_counter() - t
            size = os.path.getsize(path)
            P.load_graph(path, fmt, ctx=ctx)  # warm-up (context, allocator)
            best = 1e30
            for _ in range(args.reps):
                t = time.perf_counter()
                got = P.load_graph(path, fmt, ctx=ctx)
                best = min(best, time.perf_counter() - t)
            line = {"config": args.config, "format": fmt, "file_bytes": size, "n": g.n,
                    "edges": int(got.m), "save_s": round(save_s, 3),
                    "load_s": round(best, 4), "load_gb_per_s": round(size / best / 1e9, 3)}
            if ref is not None:
                data = open(path, "rb").read()
                t = time.perf_counter()
                st, rg = ref.read_graph(data, 0 if fmt == P.EDGE_LIST else 1, path)
                ref_s = time.perf_counter() - t
                eu, ev, ew = rg.edges()
                a = np.minimum(got.eu, got.ev).astype(np.int64) * g.n + np.maximum(got.eu, got.ev)
                o = np.argsort(a, kind="stable")
                b = eu.astype(np.int64) * g.n + ev
                same = st == "ok" and np.array_equal(a[o], b) and np.array_equal(
                    got.ew[o].view(np.uint64), ew.view(np.uint64))
                line.update({"reference_read_s": round(ref_s, 3),
                             "speedup": round(ref_s / best, 1), "identical": bool(same)})
            print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
