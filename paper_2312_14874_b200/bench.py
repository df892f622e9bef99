"""Drop-in for ``prefixscan.bench``: timed cases, sweeps and CSV records with
the scans running on the B200.

Contract kept from the reference harness (pkg/src/prefixscan/bench.py): the
algorithm labels, the ``CaseConfig`` / ``BenchRecord`` fields, the seeded
inputs of ``make_input`` (bench.py:106-111), CRC-32 checksums, the float
tolerance, verify-once-before-timing, one untimed warm-up then the median of
``reps`` timed calls, ``sweep`` over threads / block_len / dilation with the
input seed shared by every point, and a fixed-schema CSV.  The code here is
organised around two tables instead of branches:

* ``_ALGOS`` maps every label to a runner (the drop-in entry point it calls)
  and the block-length policy of its pass structure;
* ``_TIMERS`` maps ``CaseConfig.device`` to how one repetition is timed --
  ``"host"``: numpy arrays (the reference's calling convention, so each
  repetition includes the PCIe staging), ``perf_counter_ns``; ``"cuda"``:
  device-resident tensors, CUDA events on the current stream.

GPU additions: labels ``GPU`` (the library's own kernel
choice), ``GPU-LB`` (single-pass decoupled look-back) and ``GPU-RND``
(L2-region accumulate-scan), and two trailing CSV columns ``device`` and
``bandwidth_gbs`` (one read + one write per element over the median).

The verification oracle is numpy's sequential ``cumsum`` in the accumulator
type, rounded once to the element type -- the sums the reference's
``oracle_scan`` produces -- so a record's checksum never depends on the code
under test (pinned against the C restatement in tests/test_harness.py).
"""

from __future__ import annotations

import statistics
import time
import zlib
from dataclasses import dataclass, field, fields, replace
from typing import Callable, NamedTuple

import numpy as np

from . import _lib, simd
from .core import element_dtype, full_span, sequential_inclusive_scan
from .engine import ScanRequest, execute
from .plan import Dilation, SchemeId, default_block_len

FLOAT_RTOL = 1e-5

SINGLE_THREAD_ALGOS = ("Scalar", "SIMD", "SIMD-V1", "SIMD-V2", "SIMD-T")
# <kernel><scheme>[-P]: scheme 1 = scan-increment, 2 = accumulate-scan; -P = cache-partitioned
MULTI_THREAD_ALGOS = tuple(f"{k}{i}{p}" for p in ("", "-P") for k in ("Scalar", "SIMD") for i in "12")
GPU_ALGOS = ("GPU", "GPU-LB", "GPU-RND")
ALGORITHMS = SINGLE_THREAD_ALGOS + MULTI_THREAD_ALGOS + GPU_ALGOS
DEVICES = ("host", "cuda")

_REF_COLUMNS = ("algo", "elem_type", "n", "threads", "block_len", "d0", "d_last", "out_of_place", "reps",
                "median_ns", "throughput_eps", "checksum")
CSV_COLUMNS = _REF_COLUMNS + ("device", "bandwidth_gbs")


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
        problems = [msg for bad, msg in (
            (self.algo not in ALGORITHMS, f"unknown algorithm {self.algo!r}; expected one of {ALGORITHMS}"),
            (self.reps < 5, "reps must be >= 5 (median needs a stable sample)"),
            (self.device not in DEVICES, f"unknown device {self.device!r}; expected one of {DEVICES}"),
            (self.n < 0, "n must be >= 0"),
        ) if bad]
        if problems:
            raise ValueError(problems[0])
        element_dtype(self.elem_type)


def default_case_elements(threads: int) -> int:
    """Default input size: 2^24 elements for each thread up to 8 threads."""
    return (1 << 24) * min(max(threads, 1), 8)


# CSV rendering per column: floats keep their repr (round-trippable), booleans are 0/1
_CELL = {"d0": repr, "d_last": repr, "throughput_eps": repr, "bandwidth_gbs": repr,
         "out_of_place": lambda v: str(int(v))}


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
        return ",".join(_CELL.get(col, str)(getattr(self, col)) for col in CSV_COLUMNS)


def make_input(elem_type: str, n: int, seed: int) -> np.ndarray:
    """Seeded data in the reference's draws: uint32 over the whole range for
    "i32", float32 in [0, 1) for "f32"."""
    gen = np.random.default_rng(seed)
    if element_dtype(elem_type) == np.uint32:
        return gen.integers(0, 1 << 32, n, dtype=np.uint32)
    return gen.random(n, dtype=np.float32)


def checksum(buf) -> int:
    """CRC-32 over the result's bytes in C order."""
    return zlib.crc32(memoryview(np.ascontiguousarray(buf)).cast("B"))


_ACC = {np.dtype(np.uint32): np.uint64, np.dtype(np.float32): np.float64}


def oracle_scan(data: np.ndarray) -> np.ndarray:
    """Sequential inclusive sums in the accumulator type (uint64 / float64),
    rounded once to the element type: uint32 wraps mod 2^32, float32 rounds
    each running double -- the reference's _scan_kernel (core.py:86-92)."""
    acc = _ACC.get(data.dtype)
    if acc is None:
        raise ValueError(f"unsupported element dtype {data.dtype}")
    return np.cumsum(data, dtype=acc).astype(data.dtype)


def verify_output(got: np.ndarray, expected: np.ndarray, elem_type: str) -> None:
    """Integers must match exactly; floats within FLOAT_RTOL per element."""
    got, expected = np.asarray(got), np.asarray(expected)
    if element_dtype(elem_type) == np.uint32:
        diff = got != expected
        if diff.any():
            raise BenchError(f"integer output mismatch at index {int(np.argmax(diff))}")
        return
    if not got.size:
        return
    ref = expected.astype(np.float64)
    denom = np.maximum(np.abs(ref), 1e-30)
    worst = float(np.max(np.abs(got.astype(np.float64) - ref) / denom))
    if worst > FLOAT_RTOL:
        raise BenchError(f"float output off by {worst:.3e} relative (> {FLOAT_RTOL})")


# ---- the algorithm table -------------------------------------------------------------------------

class _Algo(NamedTuple):
    run: Callable      # (cfg, data, out, block_len) -> total
    blocks: str        # "none": one pass, block_len ignored; "partitioned": default if unset; "any": as given


def _plain(cfg, data, out, block_len):
    if out is None:
        return sequential_inclusive_scan(data, full_span(data))
    out[:] = data
    return sequential_inclusive_scan(out, full_span(out))


def _pinned_kernel(k: int):
    """A GPU label: the library's 1-D kernel pinned for the duration of the call."""
    def run(cfg, data, out, block_len):
        lib = _lib.load()
        saved = lib.ps_get_tuning(b"scan_kernel")
        _lib.check(lib.ps_set_tuning(b"scan_kernel", k), "ps_set_tuning")
        try:
            return _plain(cfg, data, out, block_len)
        finally:
            lib.ps_set_tuning(b"scan_kernel", saved)
    return run


def _horizontal(cfg, data, out, block_len):
    return simd.horizontal_scan(data, full_span(data), 0, cfg.lane_width, out=out)


def _vertical(scan_in_pass1: bool):
    def run(cfg, data, out, block_len):
        return simd.vertical_scan(data, full_span(data), 0, cfg.lane_width, scan_in_pass1, block_len, out=out)
    return run


def _tree(cfg, data, out, block_len):
    return simd.tree_scan_auto(data, full_span(data), 0, cfg.lane_width, block_len, out=out)


def _engine(kernel: str, scheme: SchemeId):
    def run(cfg, data, out, block_len):
        return execute(ScanRequest(data=data, out=out, kernel=kernel, scheme=scheme,
                                   dilation=Dilation(cfg.d0, cfg.d_last), block_len=block_len,
                                   threads=cfg.threads, lane_width=cfg.lane_width))
    return run


def _algo_table() -> dict:
    table = {"Scalar": _Algo(_plain, "none"), "SIMD": _Algo(_horizontal, "none"),
             "SIMD-V1": _Algo(_vertical(True), "any"), "SIMD-V2": _Algo(_vertical(False), "any"),
             "SIMD-T": _Algo(_tree, "any")}
    schemes = {"1": SchemeId.SCAN_INCREMENT_PLUS_ONE, "2": SchemeId.ACCUMULATE_SCAN_PLUS_ONE}
    for label in MULTI_THREAD_ALGOS:
        base = label[:-2] if label.endswith("-P") else label
        kernel = "simd" if base.startswith("SIMD") else "scalar"
        table[label] = _Algo(_engine(kernel, schemes[base[-1]]), "partitioned" if label.endswith("-P") else "none")
    for label, k in zip(GPU_ALGOS, (0, 1, 2)):
        table[label] = _Algo(_pinned_kernel(k), "none")
    return table


_ALGOS = _algo_table()


def _resolved_block_len(cfg: CaseConfig) -> int:
    policy = _ALGOS[cfg.algo].blocks
    if policy == "none":
        return 0
    if policy == "partitioned" and cfg.block_len <= 0:
        return default_block_len(lane_width=cfg.lane_width)
    return cfg.block_len


def _run_algorithm(cfg: CaseConfig, data, out, block_len: int):
    """One scan of ``data`` (into ``out`` if given); returns the accumulator total.
    Buffers are numpy arrays (device "host") or CUDA tensors (device "cuda")."""
    return _ALGOS[cfg.algo].run(cfg, data, out, block_len)


# ---- timing strategies ---------------------------------------------------------------------------

def _host_reps(cfg: CaseConfig, base: np.ndarray, block_len: int) -> list[int]:
    out = np.empty_like(base) if cfg.out_of_place else None
    samples = []
    for _ in range(cfg.reps + 1):
        work = base.copy()  # restored outside the timed window
        t0 = time.perf_counter_ns()
        _run_algorithm(cfg, work, out, block_len)
        samples.append(time.perf_counter_ns() - t0)
    return samples[1:]  # the first repetition warms up


def _cuda_reps(cfg: CaseConfig, base: np.ndarray, block_len: int) -> list[int]:
    import torch

    src = _device_copy(base)
    work = torch.empty_like(src)
    out = torch.empty_like(src) if cfg.out_of_place else None
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    samples = []
    for _ in range(cfg.reps + 1):
        work.copy_(src)
        torch.cuda.synchronize()
        start.record()
        _run_algorithm(cfg, work, out, block_len)
        stop.record()
        stop.synchronize()
        samples.append(round(start.elapsed_time(stop) * 1e6))
    return samples[1:]


_TIMERS = {"host": _host_reps, "cuda": _cuda_reps}


def _device_copy(base: np.ndarray):
    import torch

    if not torch.cuda.is_available():
        raise BenchError("device 'cuda' requested but no CUDA device is visible")
    return torch.from_numpy(base).cuda()


def _as_numpy(buf) -> np.ndarray:
    return buf if isinstance(buf, np.ndarray) else buf.cpu().numpy()


def _checked_result(cfg: CaseConfig, base: np.ndarray, block_len: int) -> int:
    """Run once on fresh buffers, verify against the oracle, return the CRC."""
    if cfg.device == "cuda":
        import torch
        work = _device_copy(base)
        out = torch.empty_like(work) if cfg.out_of_place else None
    else:
        work = base.copy()
        out = np.empty_like(base) if cfg.out_of_place else None
    _run_algorithm(cfg, work, out, block_len)
    result = _as_numpy(work if out is None else out)
    expected = oracle_scan(base) if cfg.n else base.copy()
    verify_output(result, expected, cfg.elem_type)
    return checksum(result)


def run_case(cfg: CaseConfig) -> BenchRecord:
    """Verify one configuration against the oracle, then time it (median of
    ``reps`` repetitions after an untimed warm-up; inputs restored outside
    the timed window)."""
    block_len = _resolved_block_len(cfg)
    base = make_input(cfg.elem_type, cfg.n, cfg.seed)
    crc = _checked_result(cfg, base, block_len)
    times = _TIMERS[cfg.device](cfg, base, block_len)
    med = int(statistics.median(times))
    moved = 2 * cfg.n * base.dtype.itemsize
    rate = (cfg.n * 1e9 / med) if (med > 0 and cfg.n) else 0.0
    gbs = (moved / med) if (med > 0 and cfg.n) else 0.0
    shared = {f.name: getattr(cfg, f.name) for f in fields(BenchRecord) if hasattr(cfg, f.name)}
    shared["block_len"] = block_len
    return BenchRecord(**shared, rep_times_ns=times, median_ns=med, throughput_eps=rate, checksum=crc,
                       bandwidth_gbs=gbs)


# sweep dimension -> (CaseConfig field it varies, value conversion)
_SWEEP_AXES = {"threads": ("threads", int), "block_len": ("block_len", int), "dilation": ("d0", float)}


def sweep(dimension: str, grid, base: CaseConfig):
    """Run ``base`` at every grid value along one dimension.  Returns
    ``(records, failures)``; a failing point is recorded as ``(value, error)``
    and the sweep goes on.  Every point keeps ``base.seed`` (same data)."""
    axis = _SWEEP_AXES.get(dimension)
    if axis is None:
        raise ValueError(f"unknown sweep dimension {dimension!r}")
    points = list(grid)
    if not points:
        raise ValueError("empty sweep grid")
    name, conv = axis
    records, failures = [], []
    for value in points:
        try:
            records.append(run_case(replace(base, **{name: conv(value)})))
        except Exception as exc:  # noqa: BLE001 - a failed point is data, not a crash
            failures.append((value, exc))
    return records, failures


def write_csv(records, fh) -> None:
    """Header plus one row per record, '\\n' line endings."""
    fh.write("\n".join([",".join(CSV_COLUMNS)] + [r.csv_row() for r in records]) + "\n")
