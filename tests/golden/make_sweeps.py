"""Golden vectors for the Blelloch step functions, produced by running the
UNMODIFIED reference (simd.up_sweep / simd.down_sweep, simd.py:356-367):

    NUMBA_CACHE_DIR=/tmp/numba_ref PYTHONPATH=/root/reference/pkg/src \\
        python tests/golden/make_sweeps.py

Writes tests/golden/sweeps.npz: for every case the input, the array after
up_sweep, the returned root, and the array after a following down_sweep.
"""

from __future__ import annotations

import os

import numpy as np

from prefixscan import simd
from prefixscan.core import Span

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    r = np.random.default_rng(2312)
    out = {}
    k = 0
    for dt in (np.uint32, np.float32, np.int64, np.float64):
        for lg in (0, 1, 3, 5, 10, 11, 12, 13, 14):
            n = 1 << lg
            if np.dtype(dt).kind == "f":
                a = r.standard_normal(n).astype(dt) * dt(1000)
            elif dt == np.uint32:
                a = r.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)  # wraps
            else:
                a = r.integers(-(1 << 40), 1 << 40, n, dtype=np.int64)
            # a span inside a larger buffer (start offset 3) to pin the span handling
            buf = np.concatenate([np.zeros(3, dt), a, np.ones(2, dt)]).astype(dt)
            up = buf.copy()
            root = simd.up_sweep(up, Span(3, n))
            down = up.copy()
            simd.down_sweep(down, Span(3, n))
            out[f"c{k}_in"] = buf
            out[f"c{k}_up"] = up
            out[f"c{k}_root"] = np.array([root], dtype=dt)
            out[f"c{k}_down"] = down
            k += 1
    np.savez_compressed(os.path.join(HERE, "sweeps.npz"), n_cases=np.array([k]), **out)
    print(f"{k} cases")


if __name__ == "__main__":
    main()
