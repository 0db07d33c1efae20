"""Shared fixtures.  `gpu`-marked tests need a B200 (run via gpurun); the rest
run on CPU and cover the oracle, golden vectors, host logic and the C ABI's
exported symbols."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the native library")


@pytest.fixture(scope="session")
def orc():
    from oracle.oracle import Restatement
    return Restatement()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import Reference, available_reference
    if not available_reference():
        pytest.skip("oracle/_ref not built (reference sources absent at build time)")
    return Reference()


@pytest.fixture(scope="session")
def pcal():
    import paper_1810_03930_b200 as P
    P.lib()  # fail loudly if the native library is missing
    return P


def rel(a, b):
    a, b = np.asarray(a, dtype=float), np.asarray(b, dtype=float)
    d = np.linalg.norm(a - b)
    s = max(np.linalg.norm(b), 1e-300)
    return d / s
