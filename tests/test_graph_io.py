"""Graph ingestion (include/psp/graph_io.hpp): the GPU text parser and the
host writer against the reference build -- graphs, ParseError messages and
line numbers, written bytes -- plus the reference's own test_graph.cpp cases.
"""
import os

import numpy as np
import pytest

import paper_1503_07192_b200 as P
from paper_1503_07192_b200 import graphs


def canon(n, eu, ev, ew):
    """(n, edges as sorted (min, max, weight bits)) -- Graph::edge_list order."""
    a = np.minimum(eu, ev).astype(np.int64)
    b = np.maximum(eu, ev).astype(np.int64)
    o = np.lexsort((b, a))
    return int(n), a[o], b[o], np.asarray(ew, np.float64)[o].view(np.uint64)


def same_graph(g, rg):
    x = canon(g.n, g.eu, g.ev, g.ew)
    y = canon(rg.n, *rg.edges())
    return x[0] == y[0] and all(np.array_equal(p, q) for p, q in zip(x[1:], y[1:]))


def ref_outcome(ref, text, fmt, name="<stream>"):
    return ref.read_graph(text, 0 if fmt == P.EDGE_LIST else 1, name)


def gpu_outcome(text, fmt, ctx, name="<stream>"):
    try:
        return "ok", P.read_graph(text, fmt, name, ctx=ctx)
    except P.ParseError as e:
        return "parse", str(e), e.line
    except P.GraphInvariantError as e:
        return "graph", str(e), 0


def check_same(ref, text, fmt, ctx):
    want = ref_outcome(ref, text, fmt)
    got = gpu_outcome(text, fmt, ctx)
    assert got[0] == want[0], (text[:200], got, want)
    if want[0] == "ok":
        assert same_graph(got[1], want[1]), text[:200]
    else:
        assert got[1] == want[1], (text[:200], got, want)
        if want[0] == "parse":
            assert got[2] == want[2]
    return want[0]


# ---- host writer (CPU) -------------------------------------------------------
def test_format_weight_shortest_exact():  # test_graph.cpp:209-215
    assert P.format_weight(3.0) == "3"
    assert P.format_weight(0.5) == "0.5"
    assert P.format_weight(1.0 / 1024.0) == "0.0009765625"
    awkward = 0.1 + 0.2
    assert float(P.format_weight(awkward)) == awkward
    for w in (1e16, 1e-300, 5e-324, 123456789.125, 2.0 ** 60, 0.0):
        assert float(P.format_weight(w)) == w


@pytest.mark.parametrize("fmt", [P.EDGE_LIST, P.DIMACS])
def test_write_graph_bytes_match_reference(ref, fmt):
    f = 0 if fmt == P.EDGE_LIST else 1
    cases = [ref.generate("grid", 9, 7, (0.5, 3.0), 11), ref.generate("tri", 6, 6, (1.0, 5.0), 2),
             ref.generate("grid", 3, 3, None, 0)]
    for rg in cases:
        eu, ev, ew = rg.edges()
        assert P.write_graph(P.Graph(rg.n, eu, ev, ew), fmt) == ref.write_graph(rg, f)
    # odd weights, edges given unsorted and reversed
    rng = np.random.default_rng(5)
    n = 500
    eu = rng.integers(0, n, 3000).astype(np.uint32)
    ev = rng.integers(0, n, 3000).astype(np.uint32)
    keep = eu != ev
    pairs = np.unique(np.stack([np.minimum(eu, ev), np.maximum(eu, ev)], 1)[keep], axis=0)
    rng.shuffle(pairs)
    w = rng.choice([0.0, 1e-310, 0.1, 1 / 3, 7.0, 1e22, 123.456e10], len(pairs))
    g = P.Graph(n, pairs[:, 1].copy(), pairs[:, 0].copy(), w)
    st, rg = ref.read_graph(P.write_graph(g, fmt), f)
    assert st == "ok" and same_graph(g, rg)
    assert P.write_graph(g, fmt) == ref.write_graph(rg, f)


def test_save_graph_file(ref, tmp_path):
    rg = ref.generate("tri", 5, 8, (0.25, 2.0), 3)
    eu, ev, ew = rg.edges()
    path = tmp_path / "g.txt"
    P.save_graph(P.Graph(rg.n, eu, ev, ew), str(path))
    assert path.read_text() == ref.write_graph(rg, 0)
    with pytest.raises(P.OracleIoError):
        P.save_graph(P.Graph(rg.n, eu, ev, ew), str(tmp_path / "no" / "such" / "dir.txt"))


# ---- GPU parser --------------------------------------------------------------
GOOD_EDGE = [
    "3 2\n0 1 1.5\n1 2 2\n",
    "# comment\n\n  3 2  \n0\t1\t1.5\r\n 1 2 2.0\n\n# tail\n",
    "3 2\n0 1 1.5\n1 2 2",                      # no final newline
    "2 1\n0 1 0\n", "2 1\n0 1 -0\n", "2 1\n1 0 .5\n", "2 1\n0 1 5.\n",
    "2 1\n0 1 1e3\n", "2 1\n0 1 1E-3\n", "2 1\n0 1 0.30000000000000004\n",
    "2 1\n0 1 123456789012345678901234567890\n", "2 1\n0 1 1e-320\n",
    "2 1\n0 1 0.0000000000000000000001\n", "2 1\n0 1 9007199254740993\n",
    "2 1\n0 1 00000000000000000000000001.25\n",
    "1 0\n", "0 0\n",
]
BAD_EDGE = [
    "", "\n\n", "# only comments\n", "3\n", "3 1 7\n", "x 1\n", "3 -1\n",
    "3 1\n0 1\n", "2 1\n0 1 1.0 junk\n", "3 1\n0 x 1\n", "3 1\n0 1 abc\n", "3 1\n0 3 1\n",
    "3 1\n0 1 -1\n", "3 1\n0 1 inf\n", "3 1\n0 1 nan\n", "3 1\n0 1 1e400\n",
    "3 1\n0 1 0x10\n", "3 1\n+0 1 1\n", "3 1\n0 1 +1\n",
    "3 1\n0 1 1\n1 2 1\n", "3 1\n0 1 1\n1 2 x\n", "3 1\n0 1 x\n1 2 y\n",
    "3 3\n0 1 1\n1 2 1\n", "2 1\n1 1 2.0\n", "3 2\n0 1 1\n1 0 2\n",
    "3 1\n0 99999999999999999999999 1\n", "3 1\n18446744073709551616 1 1\n",
    "3 2\n0 1 1\n\n# c\n1 2 1\n2 0 1\n",
]
GOOD_DIMACS = [
    "c comment\np sp 3 4\na 1 2 5\na 2 1 3\na 2 2 9\na 2 3 1\n",
    "p sp 3 0\n", "c x\n\np sp 2 2\na 1 2 1.5\na 2 1 1.5\n",
    "p sp 4 3\na 1 2 2\na 1 2 2\na 3 4 0.1\n", "p sp 3 2\na 1 2 -0\na 2 1 0\n",
    "p sp 3 2\na 1 2 0\na 2 1 -0\n", "px sp 3 1\nab 1 2 3\n",
]
BAD_DIMACS = [
    "", "c only\n", "a 1 2 3\np sp 3 1\n", "x\np sp 3 1\n", "p sp 3 1\np sp 3 1\n",
    "p sp 3\n", "p xx 2 1\na 1 2 1\n", "p sp 3 1\na 0 2 1\n", "p sp 3 1\na 1 4 1\n",
    "p sp 3 1\na 1 2\n", "p sp 3 1\na 1 2 -1\n", "p sp 3 2\na 1 2 1\n",
    "p sp 3 1\na 1 2 1\na 2 3 1\n", "p sp 3 1\nb 1 2 1\n", "p sp 3 1\na 1 2 inf\n",
    "p sp 3 2\na 1 2 1\nq\n",
]


@pytest.mark.gpu
@pytest.mark.parametrize("text", GOOD_EDGE + BAD_EDGE)
def test_read_edge_list_matches_reference(ref, ctx, text):
    check_same(ref, text, P.EDGE_LIST, ctx)


@pytest.mark.gpu
@pytest.mark.parametrize("text", GOOD_DIMACS + BAD_DIMACS)
def test_read_dimacs_matches_reference(ref, ctx, text):
    check_same(ref, text, P.DIMACS, ctx)


@pytest.mark.gpu
def test_reference_graph_io_cases(ref, ctx):  # test_graph.cpp:161-207
    rg = ref.generate("grid", 4, 5, (0.5, 3.0), 11)
    g = P.Graph(rg.n, *rg.edges())
    assert same_graph(P.read_graph(P.write_graph(g), ctx=ctx), rg)
    rt = ref.generate("tri", 4, 4, (1.0, 5.0), 2)
    gt = P.Graph(rt.n, *rt.edges())
    assert same_graph(P.read_graph(P.write_graph(gt, P.DIMACS), P.DIMACS, ctx=ctx), rt)
    m = P.read_graph("c comment\np sp 3 4\na 1 2 5\na 2 1 3\na 2 2 9\na 2 3 1\n", P.DIMACS, ctx=ctx)
    assert m.n == 3 and m.m == 2
    assert m.eu.tolist() == [0, 1] and m.ev.tolist() == [1, 2] and m.ew.tolist() == [3.0, 1.0]
    with pytest.raises(P.ParseError) as e:
        P.read_graph("2 1\n0 1 1.0 junk\n", ctx=ctx)
    assert e.value.line == 2
    with pytest.raises(P.ParseError):
        P.read_graph("2 1\n1 1 2.0\n", ctx=ctx)


@pytest.mark.gpu
def test_fuzzed_texts_match_reference(ref, ctx):
    """Random byte edits of valid files: same graph or same error."""
    rng = np.random.default_rng(17)
    base_e = P.write_graph(P.generate_grid(5, 6, (0.5, 4.0), 1))
    base_d = P.write_graph(P.generate_triangulated_grid(4, 5, (1.0, 3.0), 2), P.DIMACS)
    alphabet = list("0123456789 \t\n\r.-+eEx#cpa")
    kinds = {}
    for trial in range(400):
        fmt, base = (P.EDGE_LIST, base_e) if trial % 2 == 0 else (P.DIMACS, base_d)
        t = list(base)
        for _ in range(int(rng.integers(1, 4))):
            op = rng.integers(0, 3)
            i = int(rng.integers(0, len(t) + 1))
            if op == 0 and t:
                del t[min(i, len(t) - 1)]
            elif op == 1:
                t.insert(i, alphabet[int(rng.integers(0, len(alphabet)))])
            elif t:
                t[min(i, len(t) - 1)] = alphabet[int(rng.integers(0, len(alphabet)))]
        k = check_same(ref, "".join(t), fmt, ctx)
        kinds[k] = kinds.get(k, 0) + 1
    assert kinds.get("ok", 0) > 20 and kinds.get("parse", 0) > 100


@pytest.mark.gpu
def test_load_graph_file_round_trip(ref, ctx, tmp_path):
    g = graphs.delaunay(20_000, 9)
    for fmt in (P.EDGE_LIST, P.DIMACS):
        path = tmp_path / f"d.{fmt}"
        P.save_graph(g, str(path), fmt)
        got = P.load_graph(str(path), fmt, ctx=ctx)
        x, y = canon(got.n, got.eu, got.ev, got.ew), canon(g.n, g.eu, g.ev, g.ew)
        assert x[0] == y[0] and all(np.array_equal(p, q) for p, q in zip(x[1:], y[1:]))
        st, rg = ref.read_graph(path.read_bytes(), 0 if fmt == P.EDGE_LIST else 1, str(path))
        assert st == "ok" and same_graph(got, rg)
    with pytest.raises(P.OracleIoError) as e:
        P.load_graph(str(tmp_path / "missing.txt"), ctx=ctx)
    assert str(e.value) == f"cannot open '{tmp_path / 'missing.txt'}' for reading"
    # parse errors name the file
    bad = tmp_path / "bad.txt"
    bad.write_text("3 1\n0 1 1\n1 2 1\n")
    with pytest.raises(P.ParseError) as e:
        P.load_graph(str(bad), ctx=ctx)
    assert str(e.value) == f"{bad}:3: more edges than declared in header"


# ---- the device weight conversion, checked on the host ----------------------
def test_decimal_parse_matches_from_chars(tmp_path):
    """decimal_parse.cuh (Eisel-Lemire, __host__ __device__) against
    std::from_chars -- the reference's weight parser -- on random strings."""
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = tmp_path / "decimal_check"
    cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
    subprocess.run([cxx, "-O2", "-std=c++20", "-I", os.path.join(root, "paper_1503_07192_b200", "csrc"),
                    os.path.join(root, "tools", "decimal_check.cpp"), "-o", str(exe)], check=True)
    r = subprocess.run([str(exe), "1000000"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout
    assert " 0 mismatches" in r.stdout


def test_pow5_table_is_generated():
    """pow5_table.cuh is exactly what tools/gen_pow5.py produces."""
    import importlib.util
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("gen_pow5", os.path.join(root, "tools", "gen_pow5.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    vals = list(mod.entries())
    text = open(mod.OUT).read()
    for q, v in ((-342, vals[0]), (0, vals[342]), (308, vals[650]), (-1, vals[341])):
        assert f"0x{v >> 64:016x}ull, 0x{v & ((1 << 64) - 1):016x}ull," in text, q
    assert text.count("ull, 0x") == 2 * 651
