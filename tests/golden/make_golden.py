"""Generate golden vectors by running the UNMODIFIED reference package.

Run in the development container (the only place /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_ref PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden.py

It writes ``tests/golden/golden.npz`` + ``tests/golden/manifest.json``.  Every
case records the reference entry point called, its arguments, the input, the
buffer(s) after the call and the returned total, so ``tests/test_oracle.py``
can pin the C oracle and ``tests/test_parity_gpu.py`` can pin the CUDA path
without the reference being present (it is absent on the GPU box).

Sources of the cases:
* the reference's own known-answer tests (pkg/tests/test_core.py:19-166,
  pkg/tests/test_simd.py:31-208) restated as calls;
* seeded random inputs in the reference's generators (conftest.make_data,
  pkg/tests/conftest.py:13-17) and BASELINE.json's config generators at
  reduced n;
* quirk pins: uint32 wrap with un-wrapped 64-bit totals, horizontal uint32
  totals mod 2^32, int64 beyond 2^53 (float64 accumulator).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

import prefixscan as ref  # the reference, via PYTHONPATH
from prefixscan.core import Span, full_span
from prefixscan.engine import ScanRequest, execute
from prefixscan.plan import SchemeId

HERE = os.path.dirname(os.path.abspath(__file__))

cases = []
arrays = {}


def _total(t):
    """Record a returned total exactly: ints as decimal strings, floats as hex."""
    if isinstance(t, (np.floating, float)):
        return {"kind": "float", "hex": float(t).hex()}
    if isinstance(t, (np.integer, int)):
        return {"kind": "int", "dec": str(int(t))}
    raise TypeError(type(t))


def _store(a: np.ndarray) -> str:
    """Content-addressed storage: identical arrays are written once."""
    key = "a" + hashlib.sha1(a.dtype.str.encode() + repr(a.shape).encode() + a.tobytes()).hexdigest()[:16]
    arrays.setdefault(key, a.copy())
    return key


def add(op, inp, out, total, **meta):
    i = len(cases)
    rec = {"id": i, "op": op, "dtype": str(inp.dtype), "n": int(inp.shape[0]) if inp.ndim else 0,
           "in": _store(inp), "out": _store(out)}
    if total is not None:
        rec["total"] = _total(total)
    rec.update(meta)
    cases.append(rec)


def make_data(elem, n, seed):  # pkg/tests/conftest.py:13-17
    rng = np.random.default_rng(seed)
    if elem == "i32":
        return rng.integers(0, 1 << 32, n, dtype=np.uint32)
    return rng.random(n, dtype=np.float32)


def seq(data, start, length, offset):
    work = data.copy()
    t = ref.sequential_inclusive_scan(work, Span(start, length), offset)
    add("sequential_inclusive_scan", data, work, t, start=start, len=length, offset=offset)


def horiz(data, start, length, offset, w, oop=False):
    work = data.copy()
    out = np.zeros_like(data) if oop else None
    t = ref.horizontal_scan(work, Span(start, length), offset, w, out=out)
    add("horizontal_scan", data, out if oop else work, t, start=start, len=length,
        offset=offset, w=w, out_of_place=oop)


def main():
    # --- hand KATs (test_core.py / test_simd.py) ---------------------------------
    seq(np.array([1, 2, 3, 4], np.uint32), 0, 4, 0)
    seq(np.array([5, 7], np.uint32), 0, 2, 100)
    seq(np.array([0xFFFFFFFF, 1, 2], np.uint32), 0, 3, 0)
    seq(np.arange(10, dtype=np.uint32), 2, 4, 100)
    seq(np.array([9, 9], np.uint32), 1, 0, 5)
    d = np.array([1, 2, 3, 4], np.uint32)
    add("sequential_accumulate", d, d.copy(), ref.sequential_accumulate(d, full_span(d)), start=0, len=4)
    add("sequential_accumulate", d, d.copy(), ref.sequential_accumulate(d, Span(0, 0)), start=0, len=0)
    d = np.array([1, 3, 6], np.uint32)
    w_ = d.copy()
    ref.sequential_increment(w_, full_span(w_), 10)
    add("sequential_increment", d, w_, None, start=0, len=3, offset=10)
    for arr in (np.array([1, 3, 6, 10], np.uint32), np.array([42], np.uint32), np.empty(0, np.uint32)):
        w_ = arr.copy()
        last = ref.exclusive_from_inclusive(w_)
        add("exclusive_from_inclusive", arr, w_, last, identity=0)
    for w in (4, 8, 16):
        horiz(np.ones(2 * w, np.uint32), 0, 2 * w, 0, w)
    d = np.arange(1, 9, dtype=np.uint32)
    w_ = d.copy()
    t = ref.vertical_scan(w_, full_span(w_), 0, 4, True)
    add("vertical_scan", d, w_, t, start=0, len=8, offset=0, w=4, scan_in_pass1=True, block_len=0)
    d = np.ones(8, np.uint32)
    w_ = d.copy()
    t = ref.tree_scan(w_, full_span(w_), 0, w=4)
    add("tree_scan", d, w_, t, start=0, len=8, offset=0, w=4)

    # --- seeded random: every dtype x sizes x spans x offsets ----------------------
    gens = {
        "uint32": lambda n, s: make_data("i32", n, s),
        "float32": lambda n, s: make_data("f32", n, s),
        "int64": lambda n, s: np.random.default_rng(s).integers(0, 101, n, dtype=np.int64),
        "int32": lambda n, s: np.random.default_rng(s).integers(0, 256, n, dtype=np.int32),
    }
    sizes = [0, 1, 15, 16, 17, 31, 33, 1000, 4099, 65537]
    for name, gen in gens.items():
        for n in sizes:
            data = gen(n, 1000 + n)
            seq(data, 0, n, 0)
            if n > 20:
                seq(data, 7, n - 20, 3 if name != "float32" else 2.5)
            for w in (4, 8, 16):
                if n <= 1000 or w == 16:
                    horiz(data, 0, n, 0, w, oop=(w == 8))
            tot = ref.sequential_accumulate(data, full_span(data))
            add("sequential_accumulate", data, data.copy(), tot, start=0, len=n)
            if n:
                w_ = data.copy()
                ref.sequential_inclusive_scan(w_, full_span(w_))
                inc = w_.copy()
                last = ref.exclusive_from_inclusive(w_)
                add("exclusive_from_inclusive", inc, w_, last, identity=0)
            if n and n <= 4099:
                for sip in (True, False):
                    w_ = data.copy()
                    t = ref.vertical_scan(w_, full_span(w_), 0, 16, sip, 64)
                    add("vertical_scan", data, w_, t, start=0, len=n, offset=0, w=16,
                        scan_in_pass1=sip, block_len=64)
                w_ = data.copy()
                t = ref.tree_scan_auto(w_, full_span(w_), 0, 16, 0)
                add("tree_scan_auto", data, w_, t, start=0, len=n, offset=0, w=16, block_len=0)
            if n >= 16:
                w_ = data.copy()
                ref.sequential_increment(w_, Span(3, n - 5), 11)
                add("sequential_increment", data, w_, None, start=3, len=n - 5, offset=11)
            # engine schemes (engine.py:219-248), out of place
            if n and n <= 4099:
                for scheme in SchemeId:
                    for m, block in ((2, 0), (3, 64)):
                        out = np.empty_like(data)
                        t = execute(ScanRequest(data=data.copy(), out=out, kernel="scalar",
                                                scheme=scheme, block_len=block, threads=m))
                        add("engine", data, out, t, scheme=scheme.value, threads=m, block_len=block,
                            kernel="scalar")

    # --- quirk pins --------------------------------------------------------------
    big = np.array([1, 2, 3, 2**60, 2**62], np.int64)
    seq(big, 0, 5, 0)                       # float64 accumulator above 2^53
    seq(np.array([2**53 + 1, 1], np.int64), 0, 2, 0)
    seq(np.array([2**31 - 1, 1], np.int32), 0, 2, 0)  # int32 store wraps
    horiz(make_data("i32", 64, 5), 0, 64, 0, 16)      # uint32 horizontal total mod 2^32

    # --- BASELINE config generators at reduced n -------------------------
    c1 = np.random.default_rng(0).integers(0, 101, 1 << 16, dtype=np.int64)
    seq(c1, 0, c1.shape[0], 0)
    c2 = np.random.default_rng(1).random(1 << 16, dtype=np.float32)
    seq(c2, 0, c2.shape[0], 0)
    c3 = np.random.default_rng(2).integers(0, 2, 1 << 16, dtype=np.int32)
    w_ = c3.astype(np.int64)
    ref.sequential_inclusive_scan(w_, full_span(w_))
    last = ref.exclusive_from_inclusive(w_)
    add("widen_exclusive", c3, w_, last, note="astype(int64) + sequential_inclusive_scan + exclusive_from_inclusive")
    c4 = np.random.default_rng(3).integers(0, 256, (64, 256), dtype=np.int32)
    rows = c4.astype(np.int64)
    for r in range(rows.shape[0]):
        ref.horizontal_scan(rows[r], full_span(rows[r]), 0, 16)
    cases.append({"id": len(cases), "op": "rows_widen_inclusive", "dtype": "int32",
                  "in": _store(c4), "out": _store(rows),
                  "rows": 64, "cols": 256, "note": "astype(int64) + per-row horizontal_scan"})
    c5 = np.random.default_rng(4).integers(0, 1001, 1 << 16, dtype=np.int64)
    out = np.empty_like(c5)
    t = execute(ScanRequest(data=c5.copy(), out=out, kernel="scalar",
                            scheme=SchemeId.ACCUMULATE_SCAN_EQUAL, block_len=0, threads=4))
    add("engine", c5, out, t, scheme="accumulate-scan", threads=4, block_len=0, kernel="scalar")

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "manifest.json"), "w") as fh:
        json.dump({"generator": "tests/golden/make_golden.py", "reference": "pkg/src/prefixscan",
                   "numpy": np.__version__, "cases": cases}, fh, indent=0)
    print(f"{len(cases)} cases", file=sys.stderr)


if __name__ == "__main__":
    main()
