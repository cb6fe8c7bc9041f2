"""The reference's OWN unit tests (proj/tests/test_{shortest_paths,oracle,
query,cluster}.cpp, compiled unmodified by oracle/Makefile `shimtests`).

* ref_*: linked against the plain reference library — pins the doctest-
  compatible header (oracle/doctest/doctest.h) on CPU.
* gpu_*: linked against the reference library with its hot-path symbols
  (apsp_dense, build_oracle, boundary_apsp, query, query_parallel_inner,
  batch_query) replaced by integration/psp_gpu_shim.cpp over libpsp_gpu.so —
  the drop-in claim, checked by the reference's own assertions on a B200.
"""
from __future__ import annotations

import os
import subprocess

import pytest

import oracle


def run_suite(path: str) -> str:
    if not os.path.exists(path):
        pytest.skip(f"{path} not built (needs /root/reference at build time)")
    r = subprocess.run([path], capture_output=True, text=True, timeout=600)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "| 0 failed |" in out, out[-4000:]
    return out


@pytest.mark.parametrize("suite", oracle.SHIM_TESTS)
def test_reference_suite_on_reference(suite):
    run_suite(os.path.join(oracle.SHIM_DIR, f"ref_{suite}"))


@pytest.mark.gpu
@pytest.mark.parametrize("suite", oracle.SHIM_TESTS)
def test_reference_suite_on_gpu_shim(suite):
    out = run_suite(os.path.join(oracle.SHIM_DIR, f"gpu_{suite}"))
    print(out.strip().splitlines()[-1])


# Deterministic values the acceptance gate prints (they depend only on
# graph, k and seed, measured on the reference build)
ACCEPTANCE_VALUES = {
    1: "0 mismatches in 18304976 ordered queries across 23 oracles",
    2: "0 mismatches in 10000 random queries on 256x256 grid, k=128 (9300 Dijkstra sources)",
    3: "0 violations in 841114 boundary pairs",
    4: "stored entries {230494, 2203498, 19195346}, log-log slope 1.5950",
    5: "mean cross-component minplus_ops {212.8, 499.0, 1072.8}, log-log slope 0.5835",
    6: "(p=4: 144000 ledger vs 144000 recounted), p=1 bytes = 0",
    7: "byte-identical (17694592 bytes); parallel inner query mismatches 0/2000",
    8: "n=1024: 13.88 <= 22.63; n=4096: 21.75 <= 32.00; n=16384: 32.28 <= 45.25;",
    10: "save/load bit-identical (140328 bytes), corrupted checksum rejected",
}


@pytest.mark.gpu
def test_reference_acceptance_on_gpu_shim():
    """proj/tests/acceptance/acceptance_main.cpp, unmodified, linked against
    the shim: every oracle it builds and every query it asks (18.3M single
    queries in criterion 1, inside its 120 s budget) runs on the B200."""
    path = os.path.join(oracle.SHIM_DIR, "gpu_acceptance")
    if not os.path.exists(path):
        pytest.skip(f"{path} not built (needs /root/reference at build time)")
    r = subprocess.run([path], capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    os.makedirs("gpurun_out", exist_ok=True)
    with open(os.path.join("gpurun_out", "acceptance_gpu.log"), "w") as f:
        f.write(out)
    print(out)
    assert r.returncode == 0, out[-4000:]
    assert "10 of 10 criteria passed" in out, out[-4000:]
    lines = {int(l.split()[2].rstrip(":")): l for l in out.splitlines()
             if l.startswith(("PASS criterion", "FAIL criterion"))}
    for crit, want in ACCEPTANCE_VALUES.items():
        assert want in lines[crit], (crit, lines[crit])


@pytest.mark.gpu
def test_shim_registry_never_serves_stale_tables():
    """tests/cpp/shim_registry_main.cpp through the shim: an Oracle read
    with load_oracle into a destroyed shim-built Oracle's storage answers
    from its own tables; 20 live oracles outlast the bounded registry."""
    path = os.path.join(oracle.SHIM_DIR, "gpu_registry")
    if not os.path.exists(path):
        pytest.skip(f"{path} not built (needs /root/reference at build time)")
    r = subprocess.run([path], capture_output=True, text=True, timeout=600)
    out = r.stdout + r.stderr
    print(out)
    assert r.returncode == 0 and "0 failed" in out, out[-4000:]
