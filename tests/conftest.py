import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the CUDA C-ABI)")


U32_MASK = 0xFFFFFFFF


def make_data(elem: str, n: int, seed: int) -> np.ndarray:
    """Seeded inputs in the reference's generator (pkg/tests/conftest.py:13-17)."""
    rng = np.random.default_rng(seed)
    if elem == "i32":
        return rng.integers(0, 1 << 32, n, dtype=np.uint32)
    return rng.random(n, dtype=np.float32)


def reference_scan(data: np.ndarray) -> np.ndarray:
    """Independent numpy oracle (pkg/tests/conftest.py:20-24), widened to int64."""
    if data.dtype == np.uint32:
        return np.cumsum(data, dtype=np.uint32)
    if data.dtype.kind in "iu":
        return np.cumsum(data, dtype=np.int64).astype(data.dtype)
    return np.cumsum(data.astype(np.float64)).astype(data.dtype)


def assert_scan_matches(got, expected, rtol=1e-5, context=""):
    """Bit-exact for integers, elementwise relative tolerance for floats
    (pkg/tests/conftest.py:43-53)."""
    got = np.asarray(got)
    expected = np.asarray(expected)
    if got.dtype.kind in "iu":
        if not np.array_equal(got, expected):
            bad = np.flatnonzero(got != expected)
            raise AssertionError(f"integer mismatch {context}: first bad index {bad[:5]}")
        return
    if got.shape[0] == 0:
        return
    e = expected.astype(np.float64)
    rel = np.abs(got.astype(np.float64) - e) / np.maximum(np.abs(e), 1e-30)
    assert rel.max() <= rtol, f"float off by {rel.max():.3e} {context}"


@pytest.fixture(scope="session")
def oracle_lib():
    from oracle import oracle

    oracle.build()
    return oracle
