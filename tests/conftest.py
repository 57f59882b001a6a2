"""Shared fixtures.  CPU tests run everywhere; tests marked ``gpu`` need a
B200 and call the CUDA product through its C-ABI (paper_2107_13887_b200/capi.py).

The oracle (oracle/) is test infrastructure: the reference itself
(oracle/_ref, built from /root/reference where present) and our plain-C
restatement (oracle/_port).  Both are built on demand when missing and the
toolchain allows it."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import pyoracle  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden", "reference_outputs.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")


def _ensure(flavour):
    if not pyoracle.available(flavour):
        try:
            pyoracle.build(flavour)
        except Exception:
            pass
    return pyoracle.available(flavour)


@pytest.fixture(scope="session")
def port():
    assert _ensure("port"), "the plain-C oracle could not be built"
    return pyoracle.Oracle("port")


@pytest.fixture(scope="session")
def ref():
    if not _ensure("ref"):
        pytest.skip("reference sources not available on this box (golden fixtures cover it)")
    return pyoracle.Oracle("ref")


@pytest.fixture(scope="session")
def oracle():
    """The strongest checker available: the reference if built, else the port
    (itself pinned to the reference by the golden fixtures)."""
    if _ensure("ref"):
        return pyoracle.Oracle("ref")
    assert _ensure("port")
    return pyoracle.Oracle("port")


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN)


@pytest.fixture(scope="session")
def gpu():
    from paper_2107_13887_b200 import capi

    return capi.Context(0)
