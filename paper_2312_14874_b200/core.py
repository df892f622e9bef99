"""Drop-in for ``prefixscan.core`` (reference: pkg/src/prefixscan/core.py).

Same names, signatures, in-place semantics and error behaviour as the
reference's scalar building blocks; the work runs on the B200 through the
C-ABI library instead of numba loops:

=================================  ==========================================
reference (core.py)                here
=================================  ==========================================
sequential_inclusive_scan :118     one scan launch (ps_scan: stream kernel
                                   >= 32 MiB, look-back kernel below)
sequential_accumulate     :129     one deterministic reduction (ps_reduce)
sequential_increment      :135     one vectorised add (ps_add_offset)
exclusive_from_inclusive  :141     gather + tile shift (ps_shift_right)
=================================  ==========================================

Buffers: a CUDA ``torch.Tensor`` is scanned where it lives (no copies).  A
numpy array (or CPU tensor) is staged through the device -- that is the
end-to-end path: the host->device copy, the kernel and the device->host copy
are pipelined in chunks (ps_scan_host) and the array is updated in place,
exactly like the reference mutates its argument.

Accumulator precision (core.py:40-48): uint32 data carries a uint64 total,
float32 a float64 total.  Signed integer data carries an exact int64 total
here; the reference's numba typing turns that total into float64, which is
identical below 2^53 and lossy above it ("Parity").
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import device as dev

ELEMENT_DTYPES = {"i32": np.dtype(np.uint32), "f32": np.dtype(np.float32)}

_U32_MASK = 0xFFFFFFFF


def element_dtype(name: str) -> np.dtype:
    """Resolve an element-type label ("i32" or "f32") to a numpy dtype."""
    if name not in ELEMENT_DTYPES:
        raise ValueError(f"unknown element type {name!r}; expected one of {sorted(ELEMENT_DTYPES)}")
    return ELEMENT_DTYPES[name]


def _np_dtype(dtype) -> np.dtype:
    if isinstance(dtype, torch.dtype):
        return np.dtype(str(dtype).replace("torch.", ""))
    return np.dtype(dtype)


def accumulator_zero(dtype):
    """Additive identity in the accumulator type for an element dtype."""
    dt = _np_dtype(dtype)
    if dt.kind == "u":
        return np.uint64(0)
    if dt.kind == "i":
        return np.int64(0)
    return np.float64(0.0)


def coerce_offset(offset, dtype):
    """Coerce a running-total seed to the accumulator type for ``dtype``."""
    dt = _np_dtype(dtype)
    if dt.kind == "u":
        return np.uint64(int(offset) & 0xFFFFFFFFFFFFFFFF)
    if dt.kind == "i":
        v = int(offset) & 0xFFFFFFFFFFFFFFFF
        return np.int64(v - (1 << 64) if v >= 1 << 63 else v)
    return np.float64(offset)


def wrap_element(total, dtype):
    """Reduce an accumulator-precision total to a single element value."""
    dt = _np_dtype(dtype)
    if dt.kind in "iu":
        bits = int(total) & ((1 << (8 * dt.itemsize)) - 1)
        return np.array([bits], dtype=np.dtype(f"u{dt.itemsize}")).view(dt)[0]
    return dt.type(total)


@dataclass(frozen=True)
class Span:
    """A contiguous run of elements: ``start`` index plus ``len`` count.

    Zero-length spans are legal; every operation treats them as a no-op.
    """

    start: int
    len: int

    def __post_init__(self):
        if self.start < 0 or self.len < 0:
            raise ValueError(f"invalid span ({self.start}, {self.len})")

    @property
    def end(self) -> int:
        return self.start + self.len

    def check(self, data) -> "Span":
        size = data.shape[0]
        if self.end > size:
            raise ValueError(f"span [{self.start}, {self.end}) exceeds buffer of {size}")
        return self


def full_span(data) -> Span:
    return Span(0, data.shape[0])


# ---- buffer plumbing -------------------------------------------------------------------------

def is_device(data) -> bool:
    return isinstance(data, torch.Tensor) and data.is_cuda


def _check_buffer(data) -> None:
    if isinstance(data, np.ndarray) or isinstance(data, torch.Tensor):
        if data.ndim != 1:
            raise ValueError(f"expected a 1-D buffer, got shape {tuple(data.shape)}")
        dev.dtype_code(data.dtype)
        return
    raise ValueError(f"unsupported buffer type {type(data).__name__}")


class DeviceView:
    """A contiguous CUDA view of ``data[span]``; host (or strided) buffers are
    staged through the device and written back on ``commit``."""

    def __init__(self, data, span: Span, *, load: bool = True):
        self.data = data
        self.span = span
        if is_device(data):
            v = data[span.start:span.end]
            self.staged = not v.is_contiguous()
            self.t = v.contiguous() if self.staged else v
        else:
            sl = data[span.start:span.end]
            host = torch.from_numpy(np.ascontiguousarray(sl)) if isinstance(data, np.ndarray) else sl.contiguous()
            self.staged = True
            device = torch.device("cuda", torch.cuda.current_device())
            self.t = host.to(device) if load else torch.empty(host.shape, dtype=host.dtype, device=device)

    def commit(self) -> None:
        if not self.staged:
            return
        if is_device(self.data):
            self.data[self.span.start:self.span.end].copy_(self.t)
        elif isinstance(self.data, np.ndarray):
            self.data[self.span.start:self.span.end] = self.t.cpu().numpy()
        else:
            self.data[self.span.start:self.span.end].copy_(self.t.cpu())


def _host_contiguous(data) -> bool:
    if isinstance(data, np.ndarray):
        return data.flags["C_CONTIGUOUS"] and data.flags["WRITEABLE"]
    return isinstance(data, torch.Tensor) and not data.is_cuda and data.is_contiguous()


def _total(t: torch.Tensor, dtype):
    return dev.total_to_python(t, dev.dtype_code(dtype))


# ---- the drop-in entry points -------------------------------------------------------------------

def scan_into(data, out, span: Span, offset=0, exclusive: bool = False):
    """Shared body of every scan entry point: dst[span] = scan(src[span]).

    ``out`` may be ``None`` (in place) or a buffer of the same length (and,
    by default, the same dtype).  Returns the accumulator-precision total."""
    _check_buffer(data)
    span.check(data)
    dst = data if out is None else out
    if out is not None:
        _check_buffer(out)
        span.check(out)
    code = dev.dtype_code(data.dtype)
    if span.len == 0:
        return dev.acc_to_python(coerce_offset(offset, data.dtype), code)
    if not is_device(data) and not is_device(dst) and _host_contiguous(data) and _host_contiguous(dst):
        src_v = data[span.start:span.end]
        dst_v = dst[span.start:span.end]
        return dev.scan_host(src_v, dst_v, exclusive=exclusive, seed=offset)
    src = DeviceView(data, span)
    tgt = src if out is None else DeviceView(dst, span, load=False)
    total = dev.scan(src.t, tgt.t, exclusive=exclusive, seed=offset)
    tgt.commit()
    return _total(total, data.dtype)


def sequential_inclusive_scan(data, span: Span, offset=0):
    """Replace ``data[span]`` with running totals seeded by ``offset``
    (core.py:118-126).  Returns the final running total (span total plus
    offset) in accumulator precision, so feeding it back as the next span's
    offset continues the scan exactly."""
    return scan_into(data, None, span, offset)


def sequential_accumulate(data, span: Span):
    """Return the span's total without writing to the buffer (core.py:129-132)."""
    _check_buffer(data)
    span.check(data)
    if span.len == 0:
        return dev.acc_to_python(accumulator_zero(data.dtype), dev.dtype_code(data.dtype))
    v = DeviceView(data, span)
    return _total(dev.reduce(v.t), data.dtype)


def sequential_increment(data, span: Span, offset) -> None:
    """Add ``offset`` to every element in the span (core.py:135-138)."""
    _check_buffer(data)
    span.check(data)
    if span.len == 0:
        return
    v = DeviceView(data, span)
    dev.add_offset(v.t, coerce_offset(offset, data.dtype))
    v.commit()


def exclusive_from_inclusive(data, identity=0):
    """Convert an inclusive scan to an exclusive one in place (core.py:141-151).

    Shifts the buffer right by one, writes the identity at index 0, and
    returns the displaced last inclusive total (as an element value).  Empty
    buffers are a no-op returning the identity."""
    _check_buffer(data)
    ident = wrap_element(coerce_offset(identity, data.dtype), data.dtype)
    if data.shape[0] == 0:
        return ident
    v = DeviceView(data, full_span(data))
    last = dev.shift_right(v.t, identity=ident)
    v.commit()
    return last.cpu().numpy()[0]
