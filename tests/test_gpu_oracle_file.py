"""PSP1 oracle files (§8f next row 1): written from device tables and read
back into device memory, checked against the reference's own save_oracle /
load_oracle (src/oracle_io.cpp:106-255) byte for byte."""
from __future__ import annotations

import os

import numpy as np
import pytest

import paper_1503_07192_b200 as P
from conftest import graph_of

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["grid2x3_k2", "grid2x3_k1", "two_squares_k2", "isolated2_k2",
                                  "grid16_k8_lattice", "tri20_k20_w0", "grid32_k32_unit"])
def test_gpu_image_is_byte_identical_to_reference(golden_small, ref, tmp_path, name):
    case = golden_small[name]
    g = graph_of(case)
    k, seed = int(case["k"]), int(case["seed"])
    o = P.build_oracle(g, k, 1, seed)
    gpu_file = tmp_path / "gpu.psp"
    o.save(str(gpu_file))
    ro = ref.graph(g.n, g.eu, g.ev, g.ew).build_oracle(k, 1, seed)
    ref_file = tmp_path / "ref.psp"
    ro.save(str(ref_file))
    assert gpu_file.read_bytes() == ref_file.read_bytes()


def test_cfg1_image_and_cross_loading(golden_cfg1, ref, tmp_path):
    case = golden_cfg1
    g = graph_of(case)
    o = P.build_oracle(g, 16, 8, 0)
    gpu_file = str(tmp_path / "cfg1_gpu.psp")
    o.save(gpu_file)
    ro = ref.graph(g.n, g.eu, g.ev, g.ew).build_oracle(16, 8, 0)
    ref_file = str(tmp_path / "cfg1_ref.psp")
    ro.save(ref_file)
    assert open(gpu_file, "rb").read() == open(ref_file, "rb").read()
    # the reference's load_oracle reads the GPU-written file
    back = ref.load_oracle(gpu_file)
    d, ops = back.batch_query(case["q_v1"], case["q_v2"], 1, with_ops=True)
    assert np.array_equal(d, case["q_dist"]) and np.array_equal(ops, case["q_ops"])
    # and the device loads the reference-written file
    od = P.load_oracle(ref_file)
    assert od.value_kind == P.VALUE_U32
    d, ops = od.batch_query(case["q_v1"], case["q_v2"], with_ops=True)
    assert np.array_equal(d, case["q_dist"]) and np.array_equal(ops, case["q_ops"])
    for c in range(16):
        assert np.array_equal(od.boundary_rows(c), ro.boundary_rows(c))


def test_f32_oracle_round_trip(tmp_path):
    rng = np.random.default_rng(2)
    g = P.generate_grid(24, 24)
    g = P.Graph(g.n, g.eu, g.ev, rng.uniform(1, 2, g.m).astype(np.float32).astype(np.float64))
    o = P.build_oracle(g, 8, 2, 0)
    assert o.value_kind == P.VALUE_F32
    f = str(tmp_path / "f32.psp")
    o.save(f)
    v1, v2 = P.random_pairs(g.n, 5000, 1)
    d = o.batch_query(v1, v2)
    # loaded as f32: the same arithmetic, bit for bit
    assert np.array_equal(d, P.load_oracle(f, value_kind=P.VALUE_F32).batch_query(v1, v2))
    # AUTO: f32 table values are dyadic, so the import computes exactly in
    # u32 fixed point (no per-addition f32 rounding): within the tolerance
    d2 = P.load_oracle(f).batch_query(v1, v2)
    assert np.allclose(d2, d, rtol=1e-5, atol=0)


def test_damaged_files_raise_the_reference_error_classes(tmp_path):
    # tests/test_oracle.cpp:188-228
    o = P.build_oracle(P.generate_grid(6, 6, (1, 9), 3), 4, 1, 0)
    good = tmp_path / "good.psp"
    o.save(str(good))
    data = bytearray(good.read_bytes())
    assert P.load_oracle(str(good)).n == 36

    def write(name, blob):
        p = tmp_path / name
        p.write_bytes(bytes(blob))
        return str(p)

    flipped = bytearray(data)
    flipped[len(data) // 2] ^= 0x40
    with pytest.raises(P.ChecksumError):
        P.load_oracle(write("flip.psp", flipped))
    crc_flip = bytearray(data)
    crc_flip[-1] ^= 1
    with pytest.raises(P.ChecksumError):
        P.load_oracle(write("crc.psp", crc_flip))
    magic = bytearray(data)
    magic[0:4] = b"XSP1"
    with pytest.raises(P.FormatVersionError):
        P.load_oracle(write("magic.psp", magic))
    version = bytearray(data)
    version[4] = 2
    with pytest.raises(P.FormatVersionError):
        P.load_oracle(write("version.psp", version))
    with pytest.raises(P.OracleIoError):
        P.load_oracle(write("trunc.psp", data[:-20]))
    with pytest.raises(P.OracleIoError):
        P.load_oracle(write("trail.psp", data + b"\0"))
    with pytest.raises(P.OracleIoError):
        P.load_oracle(str(tmp_path / "missing.psp"))


def test_streamed_load_value_kinds(ref, tmp_path):
    # the streamed loader decides the value kind from the whole table section
    # (choose_kind_tables semantics): a reference image of a graph with
    # non-dyadic f64 weights cannot be u32 -> EOVERFLOW when u32 is demanded,
    # f32 within 1e-5 of the reference otherwise; a dyadic (1/1024-lattice)
    # one loads as exact u32 at q > 0 (the second conversion pass)
    rng = np.random.default_rng(4)
    g0 = P.generate_grid(20, 20)
    v1, v2 = P.random_pairs(g0.n, 4000, 5)
    for weights, want_kind in ((rng.uniform(1, 2, g0.m), P.VALUE_F32),
                               (np.round(rng.uniform(1, 2, g0.m) * 1024) / 1024, P.VALUE_U32)):
        g = P.Graph(g0.n, g0.eu, g0.ev, weights)
        ro = ref.graph(g.n, g.eu, g.ev, g.ew).build_oracle(6, 1, 0)
        f = str(tmp_path / f"kind{want_kind}.psp")
        ro.save(f)
        truth = ro.batch_query(v1, v2, 1)
        od = P.load_oracle(f)
        assert od.value_kind == want_kind
        d = od.batch_query(v1, v2)
        if want_kind == P.VALUE_U32:
            assert od.fixed_point_shift > 0
            assert np.array_equal(d, truth)
        else:
            assert np.allclose(d, truth, rtol=1e-5, atol=0)
            with pytest.raises(P.PspValueError):
                P.load_oracle(f, value_kind=P.VALUE_U32)
