"""Device-level scan API over CUDA tensors (the layer the reference-shaped
modules core / simd / engine call).

Every function here is one or two launches of the sm_100a library on the
caller's current CUDA stream and returns without synchronising; totals come
back as 1-element device tensors in the accumulator dtype (int64 for signed
input, uint64 for uint32 input, float64 for floating input -- the
accumulator typing of core.py:40-48, with signed integers kept exact instead
of numba's float64).

Look-back scratch is cached per (device, stream) and reused with epoch tags,
so steady-state calls allocate nothing and memset nothing.
"""

from __future__ import annotations

import ctypes
import struct
import threading

import numpy as np
import torch

from . import _lib

# torch / numpy dtype -> C-ABI code
_TORCH_CODES = {
    torch.int32: 1, torch.int64: 2, torch.uint32: 3, torch.uint64: 4, torch.float32: 5, torch.float64: 6,
}
_NP_CODES = {
    np.dtype(np.int32): 1, np.dtype(np.int64): 2, np.dtype(np.uint32): 3, np.dtype(np.uint64): 4,
    np.dtype(np.float32): 5, np.dtype(np.float64): 6,
}
_ACC_TORCH = {1: torch.int64, 2: torch.int64, 3: torch.uint64, 4: torch.uint64, 5: torch.float64, 6: torch.float64}
_ELEM_BYTES = {1: 4, 2: 8, 3: 4, 4: 8, 5: 4, 6: 8}


def dtype_code(dt) -> int:
    if isinstance(dt, torch.dtype):
        code = _TORCH_CODES.get(dt)
    else:
        code = _NP_CODES.get(np.dtype(dt))
    if code is None:
        raise ValueError(f"unsupported element dtype {dt}; expected one of int32, int64, uint32, "
                         "uint64, float32, float64")
    return code


def acc_dtype(dt) -> torch.dtype:
    return _ACC_TORCH[dtype_code(dt)]


def acc_bits(value, code: int) -> int:
    """Host scalar -> 8-byte accumulator bits (coerce_offset, core.py:40-48)."""
    if code in (5, 6):
        return struct.unpack("<Q", struct.pack("<d", float(value)))[0]
    return int(value) & 0xFFFFFFFFFFFFFFFF


def elem_bits(value, code: int) -> int:
    """Host scalar -> element bits (wrap_element, core.py:51-55)."""
    if code == 5:
        return struct.unpack("<I", struct.pack("<f", float(value)))[0]
    if code == 6:
        return struct.unpack("<Q", struct.pack("<d", float(value)))[0]
    if code in (1, 3):
        return int(value) & 0xFFFFFFFF
    return int(value) & 0xFFFFFFFFFFFFFFFF


_PAIR_OK: dict = {}


def _pair_ok(lib, ci: int, co: int) -> bool:
    ok = _PAIR_OK.get((ci, co))
    if ok is None:
        ok = _PAIR_OK[(ci, co)] = bool(lib.ps_pair_supported(ci, co))
    return ok


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def _stream_ptr(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _require_cuda(t: torch.Tensor, name: str) -> None:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")


class _Scratch:
    """Zero-initialised, epoch-tagged look-back scratch for one (device, stream)."""

    def __init__(self):
        self.buf: torch.Tensor | None = None
        self.epoch = 0
        # buffers a captured CUDA graph may still address: never returned to the
        # allocator, since every replay memsets and writes descriptors into them
        self.captured = False
        self.retired: list[torch.Tensor] = []

    def take(self, nbytes: int, n_epochs: int, device: torch.device,
             capturing: bool = False) -> tuple[int, int, int]:
        if capturing:
            # CUDA graph capture: the epoch is baked into the graph, so a replay would
            # meet the descriptors of the previous replay under the same epoch.  The
            # scratch is zeroed inside the graph instead (one memset node per launch),
            # which makes every replay start from a clean scratch.
            if self.buf is None or self.buf.numel() < nbytes:
                raise RuntimeError("scan scratch must exist before CUDA graph capture: run the same call "
                                   "once on the capture stream first (the usual warm-up)")
            self.captured = True
            self.buf[:max(nbytes, 16)].zero_()
            first = self.epoch + 1 if self.epoch + n_epochs <= _lib.PS_EPOCH_MAX else 1
            self.epoch = first + n_epochs - 1
            return self.buf.data_ptr(), self.buf.numel(), first
        if self.buf is None or self.buf.numel() < nbytes:
            size = max(nbytes, 1 << 16)
            if self.buf is not None:
                size = max(size, 2 * self.buf.numel())
                if self.captured:
                    self.retired.append(self.buf)
            self.buf = torch.zeros(size, dtype=torch.uint8, device=device)
            self.epoch = 0
        if self.epoch + n_epochs > _lib.PS_EPOCH_MAX:
            self.buf.zero_()
            self.epoch = 0
        first = self.epoch + 1
        self.epoch += n_epochs
        return self.buf.data_ptr(), self.buf.numel(), first


_scratch: dict[tuple[int, int], _Scratch] = {}
_scratch_lock = threading.Lock()


def _scratch_for(device: torch.device, nbytes: int, n_epochs: int = 1, kind: str = "lookback",
                 stream: int | None = None):
    if stream is None:
        stream = _stream_ptr(device)
    key = (device.index if device.index is not None else torch.cuda.current_device(), stream, kind)
    with _scratch_lock:
        s = _scratch.get(key)
        if s is None:
            s = _scratch[key] = _Scratch()
        return s.take(nbytes, n_epochs, device, torch.cuda.is_current_stream_capturing())


def _flat(t: torch.Tensor, name: str) -> torch.Tensor:
    if t.dim() != 1:
        raise ValueError(f"{name} must be 1-D, got shape {tuple(t.shape)}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t


def scan(x: torch.Tensor, out: torch.Tensor | None = None, *, exclusive: bool = False, seed=0,
         seed_terms: torch.Tensor | None = None, total: torch.Tensor | None = None) -> torch.Tensor:
    """out[i] = seed + sum(seed_terms) + sum(x[:i+1]) (exclusive: x[:i]).

    ``out`` defaults to ``x`` (in place).  Returns the 1-element device total
    (seed + sum(x)) in the accumulator dtype; nothing is synchronised."""
    _require_cuda(x, "x")
    _flat(x, "x")
    out = x if out is None else out
    _require_cuda(out, "out")
    _flat(out, "out")
    if out.shape != x.shape:
        raise ValueError("output buffer must match input shape")
    ci, co = dtype_code(x.dtype), dtype_code(out.dtype)
    lib = _lib.load()
    if not _pair_ok(lib, ci, co):
        raise ValueError(f"unsupported dtype pair {x.dtype} -> {out.dtype}")
    if total is None:
        total = torch.empty(1, dtype=_ACC_TORCH[ci], device=x.device)
    n_terms = 0
    if seed_terms is not None:
        _require_cuda(seed_terms, "seed_terms")
        if seed_terms.dtype != _ACC_TORCH[ci] or not seed_terms.is_contiguous():
            raise ValueError(f"seed_terms must be contiguous {_ACC_TORCH[ci]}")
        n_terms = seed_terms.numel()
    n = x.numel()
    stream = _stream_ptr(x.device)  # once per call: the small-input path is host-bound
    sptr, sbytes, epoch = _scratch_for(x.device, lib.ps_scan_scratch_bytes(n, ci, co), stream=stream)
    rc = lib.ps_scan(x.data_ptr(), out.data_ptr(), n, ci, co, int(bool(exclusive)), acc_bits(seed, ci),
                     _ptr(seed_terms), n_terms, total.data_ptr(), sptr, sbytes, epoch, stream)
    _lib.check(rc, "ps_scan")
    return total


def reduce(x: torch.Tensor, *, seed=0, seed_terms: torch.Tensor | None = None,
           total: torch.Tensor | None = None) -> torch.Tensor:
    """Read-only total: seed + sum(seed_terms) + sum(x) as a 1-element device tensor."""
    _require_cuda(x, "x")
    _flat(x, "x")
    ci = dtype_code(x.dtype)
    lib = _lib.load()
    if total is None:
        total = torch.empty(1, dtype=_ACC_TORCH[ci], device=x.device)
    n_terms = 0 if seed_terms is None else seed_terms.numel()
    sptr, sbytes, _ = _scratch_for(x.device, lib.ps_reduce_scratch_bytes(x.numel(), ci), 0, "reduce")
    rc = lib.ps_reduce(_ptr(x), x.numel(), ci, acc_bits(seed, ci), _ptr(seed_terms), n_terms, _ptr(total),
                       sptr, sbytes, _stream_ptr(x.device))
    _lib.check(rc, "ps_reduce")
    return total


def add_offset(x: torch.Tensor, delta=0, delta_terms: torch.Tensor | None = None) -> None:
    """x += delta + sum(delta_terms), in the accumulator dtype."""
    _require_cuda(x, "x")
    _flat(x, "x")
    ci = dtype_code(x.dtype)
    n_terms = 0 if delta_terms is None else delta_terms.numel()
    rc = _lib.load().ps_add_offset(_ptr(x), x.numel(), ci, acc_bits(delta, ci), _ptr(delta_terms), n_terms,
                                   _stream_ptr(x.device))
    _lib.check(rc, "ps_add_offset")


def shift_right(x: torch.Tensor, out: torch.Tensor | None = None, identity=0,
                last: torch.Tensor | None = None) -> torch.Tensor | None:
    """out[0] = identity, out[i] = x[i-1]; returns the displaced x[-1] as a
    1-element device tensor (element dtype), or None when x is empty."""
    _require_cuda(x, "x")
    _flat(x, "x")
    out = x if out is None else out
    if out.shape != x.shape or out.dtype != x.dtype:
        raise ValueError("output buffer must match input shape and dtype")
    ci = dtype_code(x.dtype)
    n = x.numel()
    if n == 0:
        return None
    if last is None:
        last = torch.empty(1, dtype=x.dtype, device=x.device)
    lib = _lib.load()
    sptr, sbytes, _ = _scratch_for(x.device, lib.ps_shift_right_scratch_bytes(n, ci), 0, "shift")
    rc = lib.ps_shift_right(_ptr(x), _ptr(out), n, ci, elem_bits(identity, ci), _ptr(last), sptr, sbytes,
                            _stream_ptr(x.device))
    _lib.check(rc, "ps_shift_right")
    return last


def publish_total(total: torch.Tensor, peer_mailboxes: torch.Tensor, rank: int, epoch: int, prev_epoch: int,
                  own_mailbox: torch.Tensor, timeout: torch.Tensor | None = None) -> None:
    """Fused shard-total exchange, producer side (ps_publish_total): store
    ``total`` (1-element accumulator tensor) into this rank's slot of every
    peer mailbox.  ``peer_mailboxes`` is a device int64 tensor of the peers'
    mailbox base addresses (2 x G slots of 16 bytes each)."""
    _require_cuda(total, "total")
    if peer_mailboxes.dtype != torch.int64 or not peer_mailboxes.is_cuda:
        raise ValueError("peer_mailboxes must be a CUDA int64 tensor of device addresses")
    rc = _lib.load().ps_publish_total(_ptr(total), _ptr(peer_mailboxes), peer_mailboxes.numel(), rank, epoch,
                                      prev_epoch, _ptr(own_mailbox), _ptr(timeout), _stream_ptr(total.device))
    _lib.check(rc, "ps_publish_total")


def scan_mailbox(x: torch.Tensor, out: torch.Tensor | None, mailbox_slots: int, n_wait: int, mail_epoch: int, *,
                 exclusive: bool = False, seed=0, timeout: torch.Tensor | None = None,
                 total: torch.Tensor | None = None, dtype=None) -> torch.Tensor:
    """Fused shard-total exchange, consumer side (ps_scan_mailbox): scan ``x``
    seeded with ``seed`` plus the totals found in the ``n_wait`` mailbox slots
    at device address ``mailbox_slots`` under ``mail_epoch``; the wait is inside
    the scan kernel.  ``x`` may be None (with ``dtype``) to only fold the
    mailbox into ``total``.  Returns the 1-element accumulator total."""
    if x is None:
        code = dtype_code(dtype)
        dev = total.device if total is not None else torch.device("cuda", torch.cuda.current_device())
        n, xo, oo, co = 0, None, None, code
    else:
        _require_cuda(x, "x")
        _flat(x, "x")
        out = x if out is None else out
        _flat(out, "out")
        code, co, dev, n, xo, oo = dtype_code(x.dtype), dtype_code(out.dtype), x.device, x.numel(), x, out
    if total is None:
        total = torch.empty(1, dtype=_ACC_TORCH[code], device=dev)
    lib = _lib.load()
    sptr, sbytes, epoch = _scratch_for(dev, lib.ps_scan_scratch_bytes(max(n, 1), code, co))
    rc = lib.ps_scan_mailbox(_ptr(xo), _ptr(oo), n, code, co, int(bool(exclusive)), acc_bits(seed, code),
                             mailbox_slots, n_wait, mail_epoch, _ptr(timeout), _ptr(total), sptr, sbytes, epoch,
                             _stream_ptr(dev))
    _lib.check(rc, "ps_scan_mailbox")
    return total


def tree_up_sweep(x: torch.Tensor) -> torch.Tensor:
    """Blelloch up-sweep of a power-of-two span in place (element-typed,
    simd.py:327-334); returns the root as a 1-element device tensor."""
    _require_cuda(x, "x")
    _flat(x, "x")
    root = torch.empty(1, dtype=x.dtype, device=x.device)
    rc = _lib.load().ps_tree_up_sweep(_ptr(x), x.numel(), dtype_code(x.dtype), _ptr(root), _stream_ptr(x.device))
    _lib.check(rc, "ps_tree_up_sweep")
    return root


def tree_down_sweep(x: torch.Tensor) -> None:
    """Blelloch down-sweep of an up-swept power-of-two span in place
    (simd.py:338-347): the span becomes its exclusive scan."""
    _require_cuda(x, "x")
    _flat(x, "x")
    rc = _lib.load().ps_tree_down_sweep(_ptr(x), x.numel(), dtype_code(x.dtype), _stream_ptr(x.device))
    _lib.check(rc, "ps_tree_down_sweep")


class stall_injection:
    """Context manager: in-kernel stall injection for stress tests (the GPU form
    of the reference's ``ScanRequest.delay_hook``, engine.py:91).  Every role
    hand-off of the look-back, rounds and rows kernels sleeps with probability
    ``prob`` (0..1) for a hashed, reproducible time in [0, ``max_ns``).
    Process-wide; restores the previous setting on exit."""

    _KEYS = (b"stall_seed", b"stall_prob", b"stall_ns")

    def __init__(self, seed: int = 1, prob: float = 0.1, max_ns: int = 20000):
        if not 0.0 <= prob <= 1.0 or max_ns < 0 or seed < 0:
            raise ValueError("stall_injection needs 0 <= prob <= 1, max_ns >= 0, seed >= 0")
        self.values = (int(seed) & 0xFFFFFFFF, int(round(prob * 1024)), int(max_ns))
        self.saved = None

    def __enter__(self):
        lib = _lib.load()
        self.saved = tuple(lib.ps_get_tuning(k) for k in self._KEYS)
        for k, v in zip(self._KEYS, self.values):
            _lib.check(lib.ps_set_tuning(k, v), "ps_set_tuning")
        return self

    def __exit__(self, *exc):
        lib = _lib.load()
        for k, v in zip(self._KEYS, self.saved):
            lib.ps_set_tuning(k, v)


_FLAG_CODES = {torch.uint8: 7, torch.bool: 7, torch.int8: 7}


def select(values: torch.Tensor, flags: torch.Tensor, out: torch.Tensor | None = None, *,
           partition: bool = False, count: torch.Tensor | None = None) -> tuple[torch.Tensor, torch.Tensor]:
    """Stream compaction (``partition=False``): ``out[:k] = values[flags != 0]``
    in order; stable partition (``partition=True``): additionally
    ``out[k:] = values[flags == 0]`` in order.  ``flags`` may be bool/uint8 or
    any 4/8-byte dtype (nonzero bits select).  Returns ``(out, count)`` with
    ``count`` a 1-element int64 device tensor (k); nothing is synchronised.
    ``out`` defaults to a new tensor of ``values``' length."""
    _require_cuda(values, "values")
    _require_cuda(flags, "flags")
    _flat(values, "values")
    _flat(flags, "flags")
    if flags.numel() != values.numel():
        raise ValueError("flags must have one entry per value")
    cv = dtype_code(values.dtype)
    cf = _FLAG_CODES.get(flags.dtype)
    if cf is None:
        cf = dtype_code(flags.dtype)
    n = values.numel()
    if out is None:
        out = torch.empty_like(values)
    _require_cuda(out, "out")
    _flat(out, "out")
    if out.dtype != values.dtype or out.numel() < n:
        raise ValueError("out must have values' dtype and at least as many elements")
    if count is None:
        count = torch.empty(1, dtype=torch.int64, device=values.device)
    lib = _lib.load()
    sptr, sbytes, epoch = _scratch_for(values.device, lib.ps_select_scratch_bytes(n), 1, "select")
    rc = lib.ps_select(_ptr(values), _ptr(flags), n, cv, cf, int(bool(partition)), _ptr(out), _ptr(count),
                       sptr, sbytes, epoch, _stream_ptr(values.device))
    _lib.check(rc, "ps_select")
    return out, count


def _rows_view(x: torch.Tensor, name: str) -> tuple[int, int, int]:
    if x.dim() != 2:
        raise ValueError(f"{name} must be 2-D (rows, cols)")
    if x.stride(1) != 1 and x.shape[1] > 1:
        raise ValueError(f"{name} rows must be contiguous")
    rows, cols = x.shape
    ld = x.stride(0) if rows > 1 else cols
    return rows, cols, ld


def scan_batched(x: torch.Tensor, out: torch.Tensor | None = None, *, exclusive: bool = False,
                 row_seeds: torch.Tensor | None = None, row_totals: torch.Tensor | None = None) -> None:
    """Independent scans of every row of a 2-D tensor (row-major, any row stride)."""
    _require_cuda(x, "x")
    out = x if out is None else out
    _require_cuda(out, "out")
    rows, cols, ld_in = _rows_view(x, "x")
    r2, c2, ld_out = _rows_view(out, "out")
    if (r2, c2) != (rows, cols):
        raise ValueError("output buffer must match input shape")
    ci, co = dtype_code(x.dtype), dtype_code(out.dtype)
    lib = _lib.load()
    if not lib.ps_pair_supported(ci, co):
        raise ValueError(f"unsupported dtype pair {x.dtype} -> {out.dtype}")
    for t, nm in ((row_seeds, "row_seeds"), (row_totals, "row_totals")):
        if t is not None and (t.dtype != _ACC_TORCH[ci] or t.numel() != rows or not t.is_contiguous()):
            raise ValueError(f"{nm} must be a contiguous {_ACC_TORCH[ci]} tensor of {rows} entries")
    sptr, sbytes, epoch = _scratch_for(x.device, lib.ps_scan_batched_scratch_bytes(rows, cols, ci, co))
    rc = lib.ps_scan_batched(_ptr(x), _ptr(out), rows, cols, ld_in, ld_out, ci, co, int(bool(exclusive)),
                             _ptr(row_seeds), _ptr(row_totals), sptr, sbytes, epoch, _stream_ptr(x.device))
    _lib.check(rc, "ps_scan_batched")


def reduce_batched(x: torch.Tensor, row_totals: torch.Tensor | None = None) -> torch.Tensor:
    _require_cuda(x, "x")
    rows, cols, ld = _rows_view(x, "x")
    ci = dtype_code(x.dtype)
    if row_totals is None:
        row_totals = torch.empty(rows, dtype=_ACC_TORCH[ci], device=x.device)
    rc = _lib.load().ps_reduce_batched(_ptr(x), rows, cols, ld, ci, _ptr(row_totals), _stream_ptr(x.device))
    _lib.check(rc, "ps_reduce_batched")
    return row_totals


def add_offset_batched(x: torch.Tensor, row_deltas: torch.Tensor) -> None:
    _require_cuda(x, "x")
    rows, cols, ld = _rows_view(x, "x")
    ci = dtype_code(x.dtype)
    if row_deltas.dtype != _ACC_TORCH[ci] or row_deltas.numel() != rows:
        raise ValueError(f"row_deltas must be {_ACC_TORCH[ci]} with {rows} entries")
    rc = _lib.load().ps_add_offset_batched(_ptr(x), rows, cols, ld, ci, _ptr(row_deltas), _stream_ptr(x.device))
    _lib.check(rc, "ps_add_offset_batched")


def scan_segmented(x: torch.Tensor, offsets: torch.Tensor, out: torch.Tensor | None = None, *,
                   exclusive: bool = False, seg_totals: torch.Tensor | None = None) -> torch.Tensor | None:
    """Scan every CSR segment x[offsets[s]:offsets[s+1]] independently."""
    _require_cuda(x, "x")
    _flat(x, "x")
    out = x if out is None else out
    _require_cuda(out, "out")
    _flat(out, "out")
    if out.shape != x.shape:
        raise ValueError("output buffer must match input shape")
    if offsets.dtype != torch.int64 or offsets.dim() != 1 or not offsets.is_cuda or not offsets.is_contiguous():
        raise ValueError("offsets must be a contiguous 1-D int64 CUDA tensor")
    nseg = offsets.numel() - 1
    if nseg < 0:
        raise ValueError("offsets needs at least one entry")
    ci, co = dtype_code(x.dtype), dtype_code(out.dtype)
    lib = _lib.load()
    if not _pair_ok(lib, ci, co):
        raise ValueError(f"unsupported dtype pair {x.dtype} -> {out.dtype}")
    if seg_totals is not None:
        _require_cuda(seg_totals, "seg_totals")
        if seg_totals.dtype != _ACC_TORCH[ci] or seg_totals.numel() != nseg or not seg_totals.is_contiguous():
            raise ValueError(f"seg_totals must be a contiguous {_ACC_TORCH[ci]} tensor with {nseg} entries")
    sptr, sbytes, epoch = _scratch_for(x.device, lib.ps_scan_segmented_scratch_bytes(x.numel(), ci, co))
    rc = lib.ps_scan_segmented(_ptr(x), _ptr(out), x.numel(), _ptr(offsets), nseg, ci, co, int(bool(exclusive)),
                               _ptr(seg_totals), sptr, sbytes, epoch, _stream_ptr(x.device))
    _lib.check(rc, "ps_scan_segmented")
    return seg_totals


def wrapped_block_total(x: torch.Tensor, w: int, seed=0) -> torch.Tensor:
    """uint32 total with every w-block summed mod 2^32 (simd.py:84-99)."""
    _require_cuda(x, "x")
    if x.dtype != torch.uint32:
        raise ValueError("wrapped block totals are defined for uint32 data only")
    total = torch.empty(1, dtype=torch.uint64, device=x.device)
    rc = _lib.load().ps_reduce_wrapped_blocks(_ptr(x), x.numel(), w, acc_bits(seed, 3), _ptr(total),
                                              _stream_ptr(x.device))
    _lib.check(rc, "ps_reduce_wrapped_blocks")
    return total


# ---- host buffers: the end-to-end entry point ---------------------------------------------------
DEFAULT_CHUNK_BYTES = 32 << 20  # measured best on PCIe Gen5 for large inputs (scripts/e2e_sweep.py)
MIN_CHUNK_BYTES = 4 << 20  # small inputs: >= 8 chunks so fill/drain stays short


class _HostWorkspace:
    """Device workspace of the host pipelines: NSLOT input/output slots plus
    epoch-tagged look-back scratch.  The scratch sits at an offset that depends
    on the slot sizes, so a call with a different layout re-zeroes the buffer:
    old slot data must never be read back as descriptors."""

    def __init__(self):
        self.buf = None
        self.epoch = 0
        self.layout = None

    def take(self, nbytes: int, n_epochs: int, layout, device: torch.device) -> int:
        if self.buf is None or self.buf.numel() < nbytes:
            self.buf = torch.zeros(nbytes, dtype=torch.uint8, device=device)
            self.epoch = 0
        elif layout != self.layout or self.epoch + n_epochs > _lib.PS_EPOCH_MAX:
            self.buf.zero_()
            self.epoch = 0
        self.layout = layout
        first = self.epoch + 1
        self.epoch += n_epochs
        return first


_host_ws: dict[int, _HostWorkspace] = {}
# one host pipeline at a time per device: the workspace (slots + scratch) and the
# library's per-device streams/bounce buffers are shared by every caller thread
_host_locks: dict[int, threading.Lock] = {}
_host_locks_guard = threading.Lock()


def _host_lock(index: int) -> threading.Lock:
    with _host_locks_guard:
        lk = _host_locks.get(index)
        if lk is None:
            lk = _host_locks[index] = threading.Lock()
        return lk


def _host_range(a) -> tuple[int, int]:
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("pinned_host needs C-contiguous arrays")
        return a.ctypes.data, a.nbytes
    if isinstance(a, torch.Tensor) and not a.is_cuda:
        if not a.is_contiguous():
            raise ValueError("pinned_host needs contiguous tensors")
        return a.data_ptr(), a.numel() * a.element_size()
    raise ValueError("pinned_host takes host numpy arrays or CPU tensors")


class pinned_host:
    """Context manager: page-lock caller-owned host arrays in place
    (cudaHostRegister through ``ps_host_register``) so the host pipelines DMA
    them directly at full PCIe rate; unregisters on exit what it registered.
    Arrays that are already page-locked are left alone."""

    def __init__(self, *arrays):
        self.ranges = [_host_range(a) for a in arrays if a is not None]
        self.done: list[int] = []

    def __enter__(self):
        lib = _lib.load()
        try:
            for ptr, nbytes in self.ranges:
                if nbytes == 0 or ptr in self.done:
                    continue
                flag = ctypes.c_int(0)
                _lib.check(lib.ps_host_register(ptr, nbytes, ctypes.byref(flag)), "ps_host_register")
                if flag.value:
                    self.done.append(ptr)
        except Exception:
            self.__exit__(None, None, None)
            raise
        return self

    def __exit__(self, *exc):
        lib = _lib.load()
        while self.done:
            lib.ps_host_unregister(self.done.pop())


def is_pinned(a) -> bool:
    """True if the host array's memory is page-locked."""
    ptr, _ = _host_range(a)
    return bool(_lib.load().ps_host_is_pinned(ptr))


def _host_pointer(a) -> tuple[int, int, int]:
    """(address, numel, dtype code) of a host numpy array or CPU tensor."""
    if isinstance(a, np.ndarray):
        if a.ndim != 1 or not a.flags["C_CONTIGUOUS"]:
            raise ValueError("host buffers must be contiguous 1-D arrays")
        return a.ctypes.data, a.shape[0], dtype_code(a.dtype)
    if isinstance(a, torch.Tensor) and not a.is_cuda:
        if a.dim() != 1 or not a.is_contiguous():
            raise ValueError("host buffers must be contiguous 1-D tensors")
        return a.data_ptr(), a.numel(), dtype_code(a.dtype)
    raise ValueError("expected a host numpy array or CPU tensor")


def scan_host(x, out=None, *, exclusive: bool = False, seed=0, chunk_elems: int | None = None,
              device: torch.device | int | None = None):
    """Scan HOST memory end to end (H2D -> scan -> D2H, pipelined in
    chunks over three streams).  ``out`` defaults to ``x`` (in place).
    Page-locked memory is DMA'd directly; pageable memory (a plain numpy
    array) is staged through the library's pinned bounce ring by host copy
    threads, overlapped with the transfers.  Thread-safe (one pipeline per
    device at a time).  Blocks; returns the accumulator-precision total as a
    Python number."""
    xp, n, ci = _host_pointer(x)
    out = x if out is None else out
    op, n2, co = _host_pointer(out)
    if n2 != n:
        raise ValueError("output buffer must match input shape")
    lib = _lib.load()
    if not lib.ps_pair_supported(ci, co):
        raise ValueError("unsupported dtype pair")
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else
                       (device if isinstance(device, int) else device.index or 0))
    if chunk_elems is None:
        # >= 8 chunks when the input allows it (pipeline fill/drain is one chunk each
        # way), but never below MIN_CHUNK_BYTES (per-copy overhead) or above the default
        eb = max(_ELEM_BYTES[ci], _ELEM_BYTES[co])
        want = min(DEFAULT_CHUNK_BYTES, max(MIN_CHUNK_BYTES, n * eb // 8))
        chunk_elems = max(want // eb, 1 << 16)
    wsb = lib.ps_scan_host_workspace_bytes(chunk_elems, ci, co)
    nep = lib.ps_scan_host_epochs(n, chunk_elems)
    with torch.cuda.device(dev), _host_lock(dev.index):
        ws = _host_ws.setdefault(dev.index, _HostWorkspace())
        epoch = ws.take(wsb, nep, ("1d", chunk_elems, ci, co), dev)
        tot = np.zeros(1, np.uint64)
        rc = lib.ps_scan_host(xp, op, n, ci, co, int(bool(exclusive)), acc_bits(seed, ci), tot.ctypes.data,
                              ws.buf.data_ptr(), ws.buf.numel(), chunk_elems, epoch, _stream_ptr(dev))
        _lib.check(rc, "ps_scan_host")
    return acc_to_python(tot.view(np.dtype(_acc_np(ci)))[0], ci)


def scan_batched_host(x, out=None, *, exclusive: bool = False, chunk_rows: int | None = None,
                      device: torch.device | int | None = None) -> None:
    """Per-row scans of a contiguous 2-D HOST array end to end: chunks of rows
    go H2D -> batched scan -> D2H, pipelined over three streams (both PCIe
    directions overlap).  ``out`` defaults to ``x`` (in place).  Blocks."""
    if isinstance(x, torch.Tensor):
        if x.is_cuda or x.dim() != 2 or not x.is_contiguous():
            raise ValueError("x must be a contiguous 2-D host tensor")
        rows, cols = x.shape
    else:
        if not isinstance(x, np.ndarray) or x.ndim != 2 or not x.flags["C_CONTIGUOUS"]:
            raise ValueError("x must be a C-contiguous 2-D numpy array")
        rows, cols = x.shape
    out = x if out is None else out
    if tuple(out.shape) != (rows, cols):
        raise ValueError("output buffer must match input shape")
    xp, _, ci = _host_pointer(x.reshape(-1))
    op, _, co = _host_pointer(out.reshape(-1))
    lib = _lib.load()
    if not lib.ps_pair_supported(ci, co):
        raise ValueError("unsupported dtype pair")
    if rows == 0 or cols == 0:
        return
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else
                       (device if isinstance(device, int) else device.index or 0))
    if chunk_rows is None:
        eb = max(_ELEM_BYTES[ci], _ELEM_BYTES[co])
        want = min(DEFAULT_CHUNK_BYTES, max(MIN_CHUNK_BYTES, rows * cols * eb // 8))
        chunk_rows = max(1, want // (cols * eb))
    chunk_rows = min(chunk_rows, rows)
    wsb = lib.ps_scan_batched_host_workspace_bytes(chunk_rows, cols, ci, co)
    nep = lib.ps_scan_host_epochs(rows, chunk_rows)
    with torch.cuda.device(dev), _host_lock(dev.index):
        ws = _host_ws.setdefault(dev.index, _HostWorkspace())
        epoch = ws.take(wsb, nep, ("rows", chunk_rows, cols, ci, co), dev)
        rc = lib.ps_scan_batched_host(xp, op, rows, cols, ci, co, int(bool(exclusive)), ws.buf.data_ptr(),
                                      ws.buf.numel(), chunk_rows, epoch, _stream_ptr(dev))
        _lib.check(rc, "ps_scan_batched_host")


def _acc_np(code: int):
    return np.float64 if code in (5, 6) else (np.uint64 if code in (3, 4) else np.int64)


def acc_to_python(v, code: int):
    if code in (5, 6):
        return float(v)
    return int(v)


def total_to_python(t: torch.Tensor, code: int):
    """1-element device accumulator -> Python scalar (synchronises)."""
    v = t.cpu()
    if v.dtype == torch.uint64:
        return int(v.view(torch.int64).item()) & 0xFFFFFFFFFFFFFFFF
    return acc_to_python(v.item(), code)
