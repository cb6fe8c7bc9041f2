"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck, ONE tool per run):

  compute-sanitizer --tool racecheck python tools/sanitize_check.py

Exercises every kernel family on BASELINE configs[0] (64x64 grid, k=16:
boundary graph of 6 tiles so FW phases 1-3 all run): K0 init, batched
component FW, boundary-graph FW, both query kernels, query-table extraction,
PSP1 save (f64 unpack + GPU CRC) and load (import). Checks the answers
against the committed reference fixture so a silent corruption also fails.
"""
import hashlib
import os
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1503_07192_b200 as P  # noqa: E402


def main():
    z = np.load(os.path.join(ROOT, "tests", "golden", "ref_cfg1.npz"))
    g = P.Graph(int(z["n"]), z["eu"], z["ev"], z["ew"])
    o = P.build_oracle(g, 16, 4, 0)
    h = hashlib.sha256()
    for c in range(16):
        h.update(o.component_table(c).tobytes())
        h.update(o.boundary_rows(c).tobytes())
    assert h.digest() == z["tables_sha256"].tobytes(), "tables differ from the reference"
    for kernel in ("grouped", "warp"):
        os.environ["PSP_QUERY_KERNEL"] = kernel
        d = o.batch_query(z["q_v1"][:2000], z["q_v2"][:2000])
        assert np.array_equal(d, z["q_dist"][:2000]), kernel
    os.environ.pop("PSP_QUERY_KERNEL")
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "cfg1.psp")
        o.save(path)
        o2 = P.load_oracle(path)
        assert np.array_equal(o2.batch_query(z["q_v1"][:500], z["q_v2"][:500]), z["q_dist"][:500])
    # f32 path (tolerance kernels)
    rng = np.random.default_rng(1)
    gf = P.Graph(g.n, g.eu, g.ev, rng.uniform(1, 2, g.m).astype(np.float32).astype(np.float64))
    of = P.build_oracle(gf, 16, 4, 0)
    assert of.value_kind == P.VALUE_F32
    of.batch_query(z["q_v1"][:500], z["q_v2"][:500])
    print("sanitize_check: ok")


if __name__ == "__main__":
    main()
