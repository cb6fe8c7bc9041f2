"""Profiling driver: build one configuration's oracle on cuda:0, then run a few
device-resident query batches (the bench's query step) so that ncu can
capture a steady-state query kernel launch, e.g.

  ncu --set full --clock-control none --import-source on \\
      --kernel-name regex:query_grouped --launch-skip 2 --launch-count 1 \\
      -o gpurun_out/qg python tools/profile_query.py --config delaunay1m_k1024

Prints the CUDA-event time per batch (without ncu that is the number to
compare; under ncu it is not a measurement).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1503_07192_b200 as P  # noqa: E402
from paper_1503_07192_b200 import graphs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="delaunay1m_k1024")
    ap.add_argument("--batch", type=int, default=0, help="pairs per batch (default: config's)")
    ap.add_argument("--batches", type=int, default=4)
    ap.add_argument("--kernel", default="auto", help="auto|grouped|cta|warp (PSP_QUERY_KERNEL)")
    args = ap.parse_args()
    if args.kernel != "auto":
        os.environ["PSP_QUERY_KERNEL"] = args.kernel
    dev = torch.device("cuda", 0)
    t0 = time.time()
    g, cfg = graphs.make(args.config)
    o = P.build_oracle(g, cfg["k"], os.cpu_count() or 8, 0)
    build_s = time.time() - t0
    batch = args.batch or cfg["queries"]
    v1, v2 = P.random_pairs(g.n, batch * args.batches, 1000)
    d1 = torch.from_numpy(v1.view(np.int32)).to(dev)
    d2 = torch.from_numpy(v2.view(np.int32)).to(dev)
    out = torch.empty(batch, dtype=torch.float64, device=dev)
    st = torch.cuda.Stream(device=dev)
    times = []
    for i in range(args.batches):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        o.batch_query_device(d1[i * batch:].data_ptr(), d2[i * batch:].data_ptr(),
                             out.data_ptr(), batch, st.cuda_stream)
        e1.record(st)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    print(json.dumps({"config": args.config, "batch": batch, "kernel": args.kernel,
                      "ms_per_batch": [round(t, 3) for t in times], "build_s": round(build_s, 2),
                      "b": o.b}))


if __name__ == "__main__":
    main()
