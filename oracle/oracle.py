"""ctypes front end of the CPU oracle (``oracle/liboracle.so``).

TEST INFRASTRUCTURE ONLY: imported by ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs, as the
checker and as the CPU baseline.  The product package
``paper_2312_14874_b200`` never imports this module.

Every function mirrors one reference entry point with numpy arrays in and out
(in place, like the reference), returning the accumulator-precision total the
reference returns:

* uint32 data  -> Python ``int`` (np.uint64 arithmetic, core.py:40-48)
* float32 data -> ``float`` (float64 accumulator)
* int32/int64  -> ``float`` (numba's float64 unification)
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

DTYPE_CODES = {
    np.dtype(np.int32): 1,
    np.dtype(np.int64): 2,
    np.dtype(np.uint32): 3,
    np.dtype(np.float32): 5,
    np.dtype(np.float64): 6,
}

# plan.py:24-37 SchemeId values -> oracle scheme codes
SCHEMES = {
    "scan-increment": 0,
    "accumulate-scan": 1,
    "scan-increment+1": 2,
    "accumulate-scan+1": 3,
}

_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so with the committed Makefile (gcc only)."""
    if force or not os.path.exists(LIB_PATH):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        vp, i64, i32, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
        sigs = {
            "or_scan": [i32, vp, vp, i64, i64, vp, vp],
            "or_accumulate": [i32, vp, i64, i64, vp],
            "or_increment": [i32, vp, i64, i64, vp],
            "or_shift_right": [i32, vp, i64, vp, vp],
            "or_horizontal": [i32, i32, vp, vp, i64, i64, vp, vp],
            "or_simd_accumulate": [i32, i32, vp, i64, i64, vp],
            "or_vertical_pass1_scan": [i32, vp, i64, i64, i32, vp, vp],
            "or_vertical_pass1_accumulate": [i32, vp, i64, i64, i32, vp],
            "or_vertical_pass2_increment": [i32, vp, i64, i64, i32, vp],
            "or_vertical_pass2_scan": [i32, vp, i64, i64, i32, vp],
            "or_up_sweep": [i32, vp, i64, i64, vp],
            "or_down_sweep": [i32, vp, i64, i64],
            "or_add_back": [i32, vp, vp, i64, i64, vp],
            "or_scan_widen_i32_i64": [vp, vp, i64, i32, dbl, vp],
            "or_engine_scan": [i32, vp, vp, i64, i32, i32, dbl, dbl, i64, i32, vp],
            "or_rows_scan_widen_i32_i64": [vp, vp, i64, i64, i64, i64, i32, i32],
        }
        for name, args in sigs.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = ctypes.c_int
        _lib = L
    return _lib


def _code(arr: np.ndarray) -> int:
    try:
        return DTYPE_CODES[arr.dtype]
    except KeyError:
        raise ValueError(f"oracle has no kernel for dtype {arr.dtype}") from None


def _acc_dtype(dtype) -> np.dtype:
    return np.dtype(np.uint64) if np.dtype(dtype) == np.uint32 else np.dtype(np.float64)


def _acc(value, dtype) -> np.ndarray:
    """8-byte accumulator slot, coerced like core.py:40-48 coerce_offset."""
    if np.dtype(dtype) == np.uint32:
        return np.array([int(value) & 0xFFFFFFFFFFFFFFFF], np.uint64)
    if np.dtype(dtype).kind in "iu":
        # numba: uint64(offset) then float64 on the first add
        return np.array([float(np.uint64(int(value) & 0xFFFFFFFFFFFFFFFF))], np.float64)
    return np.array([float(value)], np.float64)


def _out(slot: np.ndarray):
    v = slot[0]
    return int(v) if slot.dtype == np.uint64 else float(v)


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _check(rc: int, what: str) -> None:
    if rc:
        raise ValueError(f"oracle {what} failed with code {rc}")


def scan(data: np.ndarray, start: int, length: int, offset=0, out: np.ndarray | None = None):
    """core.py:86-92 ``_scan_kernel`` (src -> dst, default in place)."""
    dst = data if out is None else out
    off, tot = _acc(offset, data.dtype), np.zeros(1, _acc_dtype(data.dtype))
    _check(lib().or_scan(_code(data), _ptr(data), _ptr(dst), start, length, _ptr(off), _ptr(tot)), "scan")
    return _out(tot)


def accumulate(data: np.ndarray, start: int, length: int):
    tot = np.zeros(1, _acc_dtype(data.dtype))
    _check(lib().or_accumulate(_code(data), _ptr(data), start, length, _ptr(tot)), "accumulate")
    return _out(tot)


def increment(data: np.ndarray, start: int, length: int, delta) -> None:
    d = _acc(delta, data.dtype)
    _check(lib().or_increment(_code(data), _ptr(data), start, length, _ptr(d)), "increment")


def exclusive_from_inclusive(data: np.ndarray, identity=0):
    """core.py:141-151 -- returns the displaced last element (element dtype)."""
    ident = np.array([identity]).astype(data.dtype)
    if data.shape[0] == 0:
        return ident[0]
    last = np.zeros(1, data.dtype)
    _check(lib().or_shift_right(_code(data), _ptr(data), data.shape[0], _ptr(ident), _ptr(last)), "shift")
    return last[0]


def horizontal(data: np.ndarray, start: int, length: int, offset=0, w: int = 16,
               out: np.ndarray | None = None):
    dst = data if out is None else out
    off, tot = _acc(offset, data.dtype), np.zeros(1, _acc_dtype(data.dtype))
    _check(lib().or_horizontal(_code(data), w, _ptr(data), _ptr(dst), start, length, _ptr(off), _ptr(tot)),
           "horizontal")
    return _out(tot)


def simd_accumulate(data: np.ndarray, start: int, length: int, w: int = 16):
    tot = np.zeros(1, _acc_dtype(data.dtype))
    _check(lib().or_simd_accumulate(_code(data), w, _ptr(data), start, length, _ptr(tot)), "simd_accumulate")
    return _out(tot)


def vertical_pass1_scan(data, start, k, w, carry, totals):
    c = _acc(carry, data.dtype)
    _check(lib().or_vertical_pass1_scan(_code(data), _ptr(data), start, k, w, _ptr(c), _ptr(totals)), "vp1s")


def vertical_pass1_accumulate(data, start, k, w, totals):
    _check(lib().or_vertical_pass1_accumulate(_code(data), _ptr(data), start, k, w, _ptr(totals)), "vp1a")


def vertical_pass2_increment(data, start, k, w, offsets):
    _check(lib().or_vertical_pass2_increment(_code(data), _ptr(data), start, k, w, _ptr(offsets)), "vp2i")


def vertical_pass2_scan(data, start, k, w, offsets):
    _check(lib().or_vertical_pass2_scan(_code(data), _ptr(data), start, k, w, _ptr(offsets)), "vp2s")


def vertical_scan(data: np.ndarray, start: int, length: int, offset=0, w: int = 16,
                  scan_in_pass1: bool = True, block_len: int = 0):
    """simd.py:271-314 driver over the restated pass kernels (in place)."""
    acc_dt = _acc_dtype(data.dtype)
    acc = _acc(offset, data.dtype)[0]
    zero = acc_dt.type(0)
    totals = np.zeros(w, acc_dt)
    pos, end = start, start + length
    step = block_len if block_len > 0 else max(length, 1)
    while pos < end:
        region_len = min(step, end - pos)
        aligned = region_len - region_len % w
        if aligned:
            k = aligned // w
            if scan_in_pass1:
                vertical_pass1_scan(data, pos, k, w, acc, totals)
                offs = np.empty_like(totals)
                a = zero
                for i in range(w):
                    offs[i] = a
                    a = a + totals[i]
                vertical_pass2_increment(data, pos, k, w, offs)
                a = zero
                for t in totals:
                    a = a + t
                acc = a
            else:
                vertical_pass1_accumulate(data, pos, k, w, totals)
                offs = np.empty_like(totals)
                a = acc
                for i in range(w):
                    offs[i] = a
                    a = a + totals[i]
                vertical_pass2_scan(data, pos, k, w, offs)
                acc = offs[-1] + totals[-1]
        tail = region_len - aligned
        if tail:
            acc = acc_dt.type(horizontal(data, pos + aligned, tail, acc, w))
        pos += region_len
    return int(acc) if acc_dt == np.uint64 else float(acc)


def up_sweep(data: np.ndarray, start: int, length: int):
    """simd.py:327-334 / :356-360: in-place up-sweep; returns the root (element dtype)."""
    root = np.zeros(1, data.dtype)
    _check(lib().or_up_sweep(_code(data), _ptr(data), start, length, _ptr(root)), "up")
    return root[0]


def down_sweep(data: np.ndarray, start: int, length: int) -> None:
    """simd.py:338-347 / :363-367: in-place down-sweep."""
    _check(lib().or_down_sweep(_code(data), _ptr(data), start, length), "down")


def tree_scan(data: np.ndarray, start: int, length: int, offset=0):
    """simd.py:375-395: up-sweep, down-sweep, add-back (in place)."""
    scratch = data[start:start + length].copy()
    root = np.zeros(1, data.dtype)
    _check(lib().or_up_sweep(_code(data), _ptr(data), start, length, _ptr(root)), "up")
    _check(lib().or_down_sweep(_code(data), _ptr(data), start, length), "down")
    off = _acc(offset, data.dtype)
    _check(lib().or_add_back(_code(data), _ptr(data), _ptr(scratch), start, length, _ptr(off)), "add_back")
    acc_dt = _acc_dtype(data.dtype)
    total = off[0] + acc_dt.type(root[0])
    return int(total) if acc_dt == np.uint64 else float(total)


def tree_scan_auto(data: np.ndarray, start: int, length: int, offset=0, w: int = 16,
                   block_len: int = 0):
    """simd.py:398-427 peeling driver."""
    acc = offset
    step = block_len if block_len > 0 else max(length, 1)
    pos, end = start, start + length
    while pos < end:
        region_end = min(pos + step, end)
        while region_end - pos >= w:
            block = w << (((region_end - pos) // w).bit_length() - 1)
            acc = tree_scan(data, pos, block, acc)
            pos += block
        tail = region_end - pos
        if tail:
            acc = horizontal(data, pos, tail, acc, w)
            pos = region_end
    if length == 0:
        return _out(_acc(offset, data.dtype))
    return acc


def engine_scan(data: np.ndarray, out: np.ndarray | None = None, threads: int = 1,
                scheme: str = "accumulate-scan+1", block_len: int = 0, simd_w: int = 0,
                d0: float = 1.0, d_last: float = 1.0):
    """engine.py:278-384 two-pass schemes on POSIX threads (the CPU baseline)."""
    dst = data if out is None else out
    tot = np.zeros(1, _acc_dtype(data.dtype))
    _check(lib().or_engine_scan(_code(data), _ptr(data), _ptr(dst), data.shape[0], threads,
                                SCHEMES[scheme], d0, d_last, block_len, simd_w, _ptr(tot)), "engine")
    return _out(tot)


def scan_widen_i32_i64(src: np.ndarray, exclusive: bool, offset: int = 0,
                       out: np.ndarray | None = None):
    """Widen int32 -> int64, reference int64 scan, optional exclusive shift.

    No reference entry point takes int32 in and int64 out; this
    is the composition the reference user would write: astype(int64), then
    sequential_inclusive_scan, then exclusive_from_inclusive (whose return is
    the total / selected count)."""
    assert src.dtype == np.int32
    dst = np.empty(src.shape[0], np.int64) if out is None else out
    tot = np.zeros(1, np.int64)
    _check(lib().or_scan_widen_i32_i64(_ptr(src), _ptr(dst), src.shape[0], int(exclusive),
                                       float(offset), _ptr(tot)), "widen")
    return dst, int(tot[0])


def rows_scan_widen_i32_i64(src: np.ndarray, threads: int = 1, simd_w: int = 0,
                            out: np.ndarray | None = None) -> np.ndarray:
    """Per-row int32 -> int64 inclusive scans (the cfg4 CPU baseline)."""
    assert src.dtype == np.int32 and src.ndim == 2
    rows, cols = src.shape
    dst = np.empty((rows, cols), np.int64) if out is None else out
    _check(lib().or_rows_scan_widen_i32_i64(_ptr(src), _ptr(dst), rows, cols, src.strides[0] // 4,
                                            dst.strides[0] // 8, threads, simd_w), "rows")
    return dst
