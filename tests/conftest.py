import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: multi-second CPU reference runs")


@pytest.fixture(scope="session")
def port():
    from pyoracle import Port
    return Port()


@pytest.fixture(scope="session")
def ref():
    from pyoracle import Reference, have_reference
    if not have_reference():
        pytest.skip("oracle/_ref/libtronref.so not built (needs /root/reference at build time)")
    return Reference()


def rel_err(got, want):
    """oracles::rel_err (proj/tests/support/oracles.cpp:144-158): ||a-b||_2/||b||_2."""
    import numpy as np
    got = np.asarray(got, dtype=float)
    want = np.asarray(want, dtype=float)
    if got.shape != want.shape:
        return float("inf")
    if want.ndim == 0:
        return abs(float(got) - float(want)) / abs(float(want)) if want != 0 else abs(float(got))
    num = float(np.sum((got - want) ** 2))
    den = float(np.sum(want ** 2))
    return float(np.sqrt(num)) if den == 0.0 else float(np.sqrt(num / den))
