"""Drop-in for ``prefixscan.engine`` (reference: pkg/src/prefixscan/engine.py).

The reference engine runs the paper's two-pass schemes on a pool of CPU
threads: pass 1 (local scans or partition totals) -> one barrier -> pass 2
(increments or seeded scans), the partition totals passed through a
double-buffered ledger (engine.py:278-344).

On one B200 that whole structure is the *inside* of a single kernel launch:
each persistent CTA's portion of a region is a "partition" held in shared
memory, its pass 1 is the reducer warps' chunk totals, the barrier + ledger
fold is the grid-wide gather of the portion totals (fixed order, so float
carries are identical on every CTA), and pass 2 is the scanner warps'
carried scan of the same shared-memory copy -- one HBM read and one write per
element, every scheme collapsing to the same single launch (stream_kernel.cuh;
small inputs use the decoupled look-back kernel).  Across GPUs the two passes are real again (see
``distributed.py``): there SchemeId selects reduce-then-scan or
scan-then-fixup.

``ScanEngine`` keeps the reference's request validation, engine/request
matching rules, error surface (worker failure -> RuntimeError chained from
the cause) and the ``RunStats`` instrumentation, extended with the GPU
launch accounting.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass, field
from typing import Callable

import numpy as np

from .core import full_span, scan_into
from .plan import Dilation, SchemeId, compute_grid
from .simd import DEFAULT_LANE_WIDTH, SUPPORTED_LANE_WIDTHS

KERNELS = ("scalar", "simd")


class ReusableBarrier:
    """Counting barrier (engine.py:42-74) for host-side orchestration code
    written against the reference; the GPU path itself never blocks on it."""

    def __init__(self, parties: int, spin_limit: int = 200):
        if parties < 1:
            raise ValueError("barrier needs at least one participant")
        self.parties = parties
        self.generation = 0
        self._arrived = 0
        self._spin = spin_limit
        self._cv = threading.Condition()

    def wait(self) -> None:
        with self._cv:
            gen = self.generation
            self._arrived += 1
            if self._arrived == self.parties:
                self._arrived = 0
                self.generation += 1
                self._cv.notify_all()
                return
        for _ in range(self._spin):
            if self.generation != gen:
                return
        with self._cv:
            self._cv.wait_for(lambda: self.generation != gen)


def _byte_range(buf) -> tuple[int, int]:
    if isinstance(buf, np.ndarray):
        lo, hi = np.byte_bounds(buf)
        return lo, hi
    start = buf.data_ptr()
    return start, start + buf.numel() * buf.element_size()


def _shares_memory(a, b) -> bool:
    if isinstance(a, np.ndarray) and isinstance(b, np.ndarray):
        return np.shares_memory(a, b)
    if type(a) is not type(b):
        return False
    (a0, a1), (b0, b1) = _byte_range(a), _byte_range(b)
    return a0 < b1 and b0 < a1


@dataclass
class ScanRequest:
    """One scan invocation (engine.py:77-106): buffers, algorithm selection,
    tuning knobs.  ``data``/``out`` may be numpy arrays (staged through the
    GPU end to end) or CUDA tensors (scanned in place on the device)."""

    data: object
    out: object = None
    kernel: str = "scalar"
    scheme: SchemeId = SchemeId.SCAN_INCREMENT_PLUS_ONE
    dilation: Dilation = field(default_factory=Dilation)
    block_len: int = 0
    threads: int = 1
    affinity: str = "none"
    lane_width: int = DEFAULT_LANE_WIDTH
    collect_stats: bool = False
    delay_hook: Callable[[int, int, str], None] | None = None

    def __post_init__(self):
        if self.kernel not in KERNELS:
            raise ValueError(f"kernel {self.kernel!r} not one of {KERNELS}")
        if self.affinity not in ("none", "compact"):
            raise ValueError(f"unknown affinity policy {self.affinity!r}")
        if self.lane_width not in SUPPORTED_LANE_WIDTHS:
            raise ValueError(f"lane width {self.lane_width} not in {SUPPORTED_LANE_WIDTHS}")
        if self.threads < 1:
            raise ValueError("threads must be >= 1")
        if self.out is not None:
            if tuple(self.out.shape) != tuple(self.data.shape) or str(self.out.dtype) != str(self.data.dtype):
                raise ValueError("output buffer must match input shape and dtype")
            if _shares_memory(self.out, self.data):
                raise ValueError("out-of-place buffers must not overlap")


@dataclass
class RunStats:
    """Per-run instrumentation (engine.py:109-128) plus GPU accounting.

    ``iterations`` / ``barrier_waits`` / ``sync_points`` / ``roles`` are the
    REFERENCE'S PLAN for this request (the same ``compute_grid``), reported so
    callers comparing schedules keep working -- the GPU does not execute it
    (``reference_plan_only`` is True to say so).  What the GPU did is
    ``kernel_launches`` and ``bytes_moved``."""

    iterations: int = 0
    barrier_waits: int = 0
    sync_points: int = 0
    roles: list = field(default_factory=list)
    kernel_launches: int = 0
    bytes_moved: int = 0
    reference_plan_only: bool = True

    def idle_pairs(self, threads: int) -> list:
        pairs = []
        for k, passes in enumerate(self.roles):
            for p, items in enumerate(passes):
                busy = {t for t, _, ln in items if ln > 0}
                pairs.extend((k, p + 1, t) for t in range(threads) if t not in busy)
        return pairs


class ScanEngine:
    """One scan at a time per engine (engine.py:149-155); executes requests
    on the current CUDA device through ``core.scan_into`` (one launch of the
    library's 1-D scan: the shared-memory-region accumulate-scan kernel for
    large inputs, the decoupled look-back kernel otherwise)."""

    def __init__(self, threads: int = 1, affinity: str = "none"):
        if threads < 1:
            raise ValueError("threads must be >= 1")
        if affinity not in ("none", "compact"):
            raise ValueError(f"unknown affinity policy {affinity!r}")
        self.threads = threads
        self.affinity = affinity
        self.barrier = ReusableBarrier(threads)
        self.last_stats: RunStats | None = None
        self._lock = threading.Lock()
        self._closed = False

    def close(self) -> None:
        self._closed = True

    def __enter__(self) -> "ScanEngine":
        return self

    def __exit__(self, *exc) -> None:
        self.close()

    def run_two_pass(self, request: ScanRequest):
        if request.block_len != 0:
            raise ValueError("two-pass execution expects block_len == 0")
        return self.run(request)

    def run_partitioned(self, request: ScanRequest):
        if request.block_len <= 0:
            raise ValueError("partitioned execution expects block_len > 0")
        return self.run(request)

    def run(self, request: ScanRequest):
        """Execute a request; returns the grand total in accumulator precision."""
        if request.threads != self.threads:
            raise ValueError(f"request wants {request.threads} threads, engine has {self.threads}")
        if request.affinity != self.affinity:
            raise ValueError(f"request wants affinity {request.affinity!r}, engine has {self.affinity!r}")
        n = request.data.shape[0]
        grid = compute_grid(n, self.threads, request.scheme, request.dilation, request.block_len,
                            request.lane_width)
        with self._lock:
            try:
                if request.delay_hook is not None:
                    request.delay_hook(0, 0, "pass1")
                total = scan_into(request.data, request.out, full_span(request.data), 0)
                if request.delay_hook is not None:
                    request.delay_hook(0, 0, "pass2")
            except ValueError:
                raise
            except BaseException as exc:
                raise RuntimeError("worker 0 failed") from exc
        if request.collect_stats:
            self.last_stats = self._stats(request, grid, n)
        return total

    @staticmethod
    def _stats(request: ScanRequest, grid, n: int) -> RunStats:
        roles = []
        for lay in grid.layouts:
            roles.append(([(it.thread, it.role, lay.spans[it.span_index].len) for it in lay.pass1],
                          [(it.thread, it.role, lay.spans[it.span_index].len) for it in lay.pass2]))
        esize = np.dtype(str(request.data.dtype).replace("torch.", "")).itemsize
        return RunStats(iterations=grid.iterations, barrier_waits=grid.iterations,
                        sync_points=grid.iterations + 1, roles=roles,
                        kernel_launches=1 if n else 0, bytes_moved=2 * n * esize)


_ENGINES: dict[tuple[int, str], ScanEngine] = {}
_ENGINES_LOCK = threading.Lock()


def shared_engine(threads: int, affinity: str = "none") -> ScanEngine:
    """Process-wide engine cache (engine.py:398-406)."""
    with _ENGINES_LOCK:
        key = (threads, affinity)
        if key not in _ENGINES:
            _ENGINES[key] = ScanEngine(threads, affinity)
        return _ENGINES[key]


def execute(request: ScanRequest):
    """Run one request on the shared engine for its thread/affinity config."""
    return shared_engine(request.threads, request.affinity).run(request)
