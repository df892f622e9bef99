"""Drop-in for ``prefixscan.bench`` (reference: pkg/src/prefixscan/bench.py).

The reference harness times one configuration at a time: seeded input,
one verification against the sequential oracle before any timing (a
benchmark of a wrong result is meaningless), a warm-up repetition, then the
median of ``reps`` timed calls, written as a fixed-schema CSV row
(bench.py:1-244).  This module keeps that contract -- the same algorithm
labels, ``CaseConfig`` / ``BenchRecord`` fields, ``make_input`` draws, CRC-32
checksum, float tolerance, ``sweep`` / ``write_csv`` behaviour -- with the
scans running on the B200 through this package's drop-in entry points.

What the GPU adds:

* ``GPU_ALGOS``: labels that name the device kernels directly -- ``GPU``
  (the library's own choice), ``GPU-LB`` (single-pass decoupled look-back,
  ``scan_kernel=1``) and ``GPU-RND`` (L2-region accumulate-scan,
  ``scan_kernel=2``).
* ``CaseConfig.device``: ``"host"`` times the reference's calling convention
  (numpy arrays in host memory, so every repetition includes the
  host->device->host staging); ``"cuda"`` times device-resident tensors with
  CUDA events (input restored outside the timed window, as the reference
  restores its input outside ``perf_counter_ns``).
* Two trailing CSV columns, ``device`` and ``bandwidth_gbs`` (algorithmic
  bytes -- one read and one write per element -- over the median time);
  readers that select the reference's columns by name are unaffected.

The verification oracle here is numpy (``np.cumsum`` in the accumulator
type, then the element type: the reference's ``oracle_scan`` computes the
same sequential sums, bench.py:116-119), so a record's checksum never
depends on the code under test.
"""

from __future__ import annotations

import contextlib
import statistics
import time
import zlib
from dataclasses import dataclass, field, replace

import numpy as np

from . import _lib, simd
from .core import element_dtype, full_span, sequential_inclusive_scan
from .engine import ScanRequest, execute
from .plan import Dilation, SchemeId, default_block_len

FLOAT_RTOL = 1e-5

CSV_COLUMNS = ("algo", "elem_type", "n", "threads", "block_len", "d0", "d_last",
               "out_of_place", "reps", "median_ns", "throughput_eps", "checksum",
               "device", "bandwidth_gbs")

SINGLE_THREAD_ALGOS = ("Scalar", "SIMD", "SIMD-V1", "SIMD-V2", "SIMD-T")
MULTI_THREAD_ALGOS = ("Scalar1", "Scalar2", "SIMD1", "SIMD2",
                      "Scalar1-P", "Scalar2-P", "SIMD1-P", "SIMD2-P")
GPU_ALGOS = ("GPU", "GPU-LB", "GPU-RND")
ALGORITHMS = SINGLE_THREAD_ALGOS + MULTI_THREAD_ALGOS + GPU_ALGOS
DEVICES = ("host", "cuda")

_MT_TABLE = {
    "Scalar1": ("scalar", SchemeId.SCAN_INCREMENT_PLUS_ONE, False),
    "Scalar2": ("scalar", SchemeId.ACCUMULATE_SCAN_PLUS_ONE, False),
    "SIMD1": ("simd", SchemeId.SCAN_INCREMENT_PLUS_ONE, False),
    "SIMD2": ("simd", SchemeId.ACCUMULATE_SCAN_PLUS_ONE, False),
    "Scalar1-P": ("scalar", SchemeId.SCAN_INCREMENT_PLUS_ONE, True),
    "Scalar2-P": ("scalar", SchemeId.ACCUMULATE_SCAN_PLUS_ONE, True),
    "SIMD1-P": ("simd", SchemeId.SCAN_INCREMENT_PLUS_ONE, True),
    "SIMD2-P": ("simd", SchemeId.ACCUMULATE_SCAN_PLUS_ONE, True),
}
# GPU label -> ps_set_tuning("scan_kernel", k): 0 = library default
_GPU_KERNEL = {"GPU": 0, "GPU-LB": 1, "GPU-RND": 2}


class BenchError(RuntimeError):
    """A case could not produce a trustworthy measurement."""


@dataclass(frozen=True)
class CaseConfig:
    """One benchmark configuration (one future CSV row)."""

    algo: str = "Scalar"
    elem_type: str = "i32"
    n: int = 1 << 20
    threads: int = 1
    block_len: int = 0  # elements per thread per iteration; 0 = unpartitioned
    d0: float = 1.0
    d_last: float = 1.0
    out_of_place: bool = False
    seed: int = 0
    reps: int = 5
    lane_width: int = simd.DEFAULT_LANE_WIDTH
    device: str = "host"

    def __post_init__(self):
        if self.algo not in ALGORITHMS:
            raise ValueError(f"unknown algorithm {self.algo!r}; expected one of {ALGORITHMS}")
        if self.reps < 5:
            raise ValueError("reps must be >= 5 (median needs a stable sample)")
        if self.device not in DEVICES:
            raise ValueError(f"unknown device {self.device!r}; expected one of {DEVICES}")
        if self.n < 0:
            raise ValueError("n must be >= 0")
        element_dtype(self.elem_type)


def default_case_elements(threads: int) -> int:
    """Desk-scale default input size: 2^24 elements per thread, 8-thread cap
    (bench.py:74-76)."""
    return (1 << 24) * max(1, min(threads, 8))


@dataclass
class BenchRecord:
    """One measured configuration with its derived throughput."""

    algo: str
    elem_type: str
    n: int
    threads: int
    block_len: int
    d0: float
    d_last: float
    out_of_place: bool
    reps: int
    rep_times_ns: list[int] = field(default_factory=list)
    median_ns: int = 0
    throughput_eps: float = 0.0
    checksum: int = 0
    device: str = "host"
    bandwidth_gbs: float = 0.0

    def csv_row(self) -> str:
        return ",".join([
            self.algo, self.elem_type, str(self.n), str(self.threads),
            str(self.block_len), repr(self.d0), repr(self.d_last),
            str(int(self.out_of_place)), str(self.reps), str(self.median_ns),
            repr(self.throughput_eps), str(self.checksum), self.device,
            repr(self.bandwidth_gbs),
        ])


def make_input(elem_type: str, n: int, seed: int) -> np.ndarray:
    """Seeded input data: uniform 32-bit ints, or floats uniform in [0, 1)
    (the reference's exact draws, bench.py:106-111)."""
    rng = np.random.default_rng(seed)
    if elem_type == "i32":
        return rng.integers(0, 1 << 32, n, dtype=np.uint32)
    return rng.random(n, dtype=np.float32)


def checksum(buf: np.ndarray) -> int:
    """CRC-32 of the result bytes (bench.py:114-115)."""
    return zlib.crc32(np.ascontiguousarray(buf).tobytes())


def oracle_scan(data: np.ndarray) -> np.ndarray:
    """Sequential inclusive scan in the accumulator type, stored in the
    element type: uint32 wraps mod 2^32, float32 sums in float64 left to
    right (np.cumsum is sequential) and rounds once per element -- what the
    reference's oracle computes (bench.py:116-119, core.py:86-92)."""
    if data.dtype == np.uint32:
        return np.cumsum(data, dtype=np.uint64).astype(np.uint32)
    if data.dtype == np.float32:
        return np.cumsum(data, dtype=np.float64).astype(np.float32)
    raise ValueError(f"unsupported element dtype {data.dtype}")


def verify_output(got: np.ndarray, expected: np.ndarray, elem_type: str) -> None:
    """Exact in integer mode; elementwise relative tolerance for floats
    (bench.py:122-136)."""
    if elem_type == "i32":
        if not np.array_equal(got, expected):
            bad = int(np.flatnonzero(got != expected)[0])
            raise BenchError(f"integer output mismatch at index {bad}")
        return
    if got.shape[0] == 0:
        return
    e = expected.astype(np.float64)
    rel = np.abs(got.astype(np.float64) - e) / np.maximum(np.abs(e), 1e-30)
    worst = float(rel.max())
    if worst > FLOAT_RTOL:
        raise BenchError(f"float output off by {worst:.3e} relative (> {FLOAT_RTOL})")


def _resolved_block_len(cfg: CaseConfig) -> int:
    name = cfg.algo
    if name in ("Scalar", "SIMD") or name in GPU_ALGOS:
        return 0  # one-pass algorithms have no second pass to localize
    if name in _MT_TABLE:
        _, _, partitioned = _MT_TABLE[name]
        if not partitioned:
            return 0
        return cfg.block_len if cfg.block_len > 0 else default_block_len(lane_width=cfg.lane_width)
    return cfg.block_len  # vertical / tree honor any block size, 0 included


@contextlib.contextmanager
def _kernel_choice(algo: str):
    """Pin the library's 1-D kernel for a GPU label, restoring it after."""
    k = _GPU_KERNEL.get(algo)
    if k is None:
        yield
        return
    lib = _lib.load()
    prev = lib.ps_get_tuning(b"scan_kernel")
    _lib.check(lib.ps_set_tuning(b"scan_kernel", k), "ps_set_tuning")
    try:
        yield
    finally:
        lib.ps_set_tuning(b"scan_kernel", prev)


def _run_algorithm(cfg: CaseConfig, data, out, block_len: int):
    """Dispatch one scan; returns the grand total (accumulator precision).
    ``data`` / ``out`` are numpy arrays (device "host") or CUDA tensors."""
    name = cfg.algo
    span = full_span(data)
    if name == "Scalar" or name in GPU_ALGOS:
        with _kernel_choice(name):
            if out is None:
                return sequential_inclusive_scan(data, span)
            out[:] = data
            return sequential_inclusive_scan(out, span)
    if name == "SIMD":
        return simd.horizontal_scan(data, span, 0, cfg.lane_width, out=out)
    if name == "SIMD-V1":
        return simd.vertical_scan(data, span, 0, cfg.lane_width, True, block_len, out=out)
    if name == "SIMD-V2":
        return simd.vertical_scan(data, span, 0, cfg.lane_width, False, block_len, out=out)
    if name == "SIMD-T":
        return simd.tree_scan_auto(data, span, 0, cfg.lane_width, block_len, out=out)
    kernel, scheme, _ = _MT_TABLE[name]
    req = ScanRequest(data=data, out=out, kernel=kernel, scheme=scheme,
                      dilation=Dilation(cfg.d0, cfg.d_last), block_len=block_len,
                      threads=cfg.threads, lane_width=cfg.lane_width)
    return execute(req)


def _to_device(base: np.ndarray):
    import torch

    if not torch.cuda.is_available():
        raise BenchError("device 'cuda' requested but no CUDA device is visible")
    return torch.from_numpy(base).cuda()


def _to_host(buf) -> np.ndarray:
    if isinstance(buf, np.ndarray):
        return buf
    return buf.cpu().numpy()


def _timed_reps(cfg: CaseConfig, base: np.ndarray, block_len: int) -> list[int]:
    """reps + 1 calls, the first a warm-up; only the scan call is timed."""
    times = []
    if cfg.device == "cuda":
        import torch

        src = _to_device(base)
        work = torch.empty_like(src)
        out = torch.empty_like(src) if cfg.out_of_place else None
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for rep in range(cfg.reps + 1):
            work.copy_(src)
            torch.cuda.synchronize()
            ev0.record()
            _run_algorithm(cfg, work, out, block_len)
            ev1.record()
            ev1.synchronize()
            if rep:
                times.append(int(round(ev0.elapsed_time(ev1) * 1e6)))
        return times
    out = np.empty_like(base) if cfg.out_of_place else None
    for rep in range(cfg.reps + 1):
        work = base.copy()
        t0 = time.perf_counter_ns()
        _run_algorithm(cfg, work, out, block_len)
        elapsed = time.perf_counter_ns() - t0
        if rep:
            times.append(elapsed)
    return times


def run_case(cfg: CaseConfig) -> BenchRecord:
    """Measure one configuration (bench.py:163-196).

    The output is verified against the oracle once before any timing; a
    failed verification aborts the case. One warm-up repetition is excluded
    from the statistics. Input copies happen outside the timed window.
    """
    block_len = _resolved_block_len(cfg)
    base = make_input(cfg.elem_type, cfg.n, cfg.seed)
    expected = oracle_scan(base) if cfg.n else base.copy()

    if cfg.device == "cuda":
        work = _to_device(base)
        import torch

        out = torch.empty_like(work) if cfg.out_of_place else None
    else:
        work = base.copy()
        out = np.empty_like(base) if cfg.out_of_place else None
    _run_algorithm(cfg, work, out, block_len)
    result = _to_host(out if cfg.out_of_place else work)
    verify_output(result, expected, cfg.elem_type)
    crc = checksum(result)

    times = _timed_reps(cfg, base, block_len)
    med = int(statistics.median(times))
    eps = cfg.n / (med / 1e9) if med > 0 and cfg.n else 0.0
    gbs = 2 * cfg.n * base.dtype.itemsize / med if med > 0 and cfg.n else 0.0
    return BenchRecord(
        algo=cfg.algo, elem_type=cfg.elem_type, n=cfg.n, threads=cfg.threads,
        block_len=block_len, d0=cfg.d0, d_last=cfg.d_last,
        out_of_place=cfg.out_of_place, reps=cfg.reps, rep_times_ns=times,
        median_ns=med, throughput_eps=eps, checksum=crc, device=cfg.device,
        bandwidth_gbs=gbs)


def sweep(dimension: str, grid, base: CaseConfig):
    """One record per grid point along a dimension; failures don't stop it
    (bench.py:199-228).

    Returns ``(records, failures)`` where failures are ``(value, error)``
    pairs. The input seed is shared across points so every point scans the
    same data.
    """
    if dimension not in ("threads", "block_len", "dilation"):
        raise ValueError(f"unknown sweep dimension {dimension!r}")
    grid = list(grid)
    if not grid:
        raise ValueError("empty sweep grid")
    records, failures = [], []
    for value in grid:
        if dimension == "threads":
            cfg = replace(base, threads=int(value))
        elif dimension == "block_len":
            cfg = replace(base, block_len=int(value))
        else:
            cfg = replace(base, d0=float(value))
        try:
            records.append(run_case(cfg))
        except Exception as exc:
            failures.append((value, exc))
    return records, failures


def write_csv(records, fh) -> None:
    """Fixed-schema CSV: one header row, one row per record, LF endings."""
    fh.write(",".join(CSV_COLUMNS) + "\n")
    for rec in records:
        fh.write(rec.csv_row() + "\n")
