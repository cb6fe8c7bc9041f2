"""Shared pytest setup.

Markers: ``gpu`` — needs a B200 (run with ``-m gpu`` on the GPU box); every
other test runs on CPU. The oracle (oracle/) is used here only as the
checker.
"""
from __future__ import annotations

import os
import sys

import numpy as np
import pytest

# torch first: its libtorch_cuda needs the NCCL it ships (2.28). The library
# dlopens "libnccl.so.2" on first multi-GPU use and binds to whichever copy
# is already loaded; were the system NCCL (2.27) loaded first, a later
# `import torch` in the same process would fail on a missing 2.28 symbol.
try:
    import torch  # noqa: F401
except ImportError:  # pragma: no cover - CPU images without torch
    pass

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")
    config.addinivalue_line("markers", "slow: long-running")


def load_small() -> dict:
    z = np.load(os.path.join(GOLDEN, "ref_small.npz"))
    cases: dict = {}
    for key in z.files:
        name, field = key.split("/", 1)
        cases.setdefault(name, {})[field] = z[key]
    return cases


@pytest.fixture(scope="session")
def golden_small() -> dict:
    return load_small()


@pytest.fixture(scope="session")
def golden_cfg1() -> dict:
    z = np.load(os.path.join(GOLDEN, "ref_cfg1.npz"))
    return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def ref():
    import oracle
    if not os.path.exists(oracle.REF_SO):
        pytest.skip("reference build oracle/_ref/libpspref.so not present")
    return oracle.RefLib()


@pytest.fixture(scope="session")
def ctx():
    import paper_1503_07192_b200 as P
    return P.default_context()


def graph_of(case: dict):
    import paper_1503_07192_b200 as P
    return P.Graph(int(case["n"]), case["eu"], case["ev"], case["ew"])
