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
