"""Drop-in for ``prefixscan.simd`` (reference: pkg/src/prefixscan/simd.py).

The reference models three CPU SIMD kernel families over a w-lane register
(w in {4, 8, 16}).  On the B200 the "register" is a 32-lane warp and a chunk
of rows per warp, so every family's *result* comes from the same 1-D scan
launch (ps_scan); what is kept per family is its public contract -- names, argument
checks, in/out-of-place behaviour and the exact returned totals:

* horizontal_scan (simd.py:134-148): for uint32 data the reference carries
  each w-block's sum out of a uint32 register, so its returned total keeps
  every block sum only mod 2^32; that total is reproduced exactly by a
  read-only wrapped-block reduction (ps_reduce_wrapped_blocks) run before
  the scan.
* vertical family (simd.py:162-321): the pass functions are batched scans
  over the w lane-chunks (ps_scan_batched with row seeds / row totals,
  ps_reduce_batched, ps_add_offset_batched); vertical_scan is one scan.
* tree family (simd.py:324-427): tree_scan / tree_scan_auto are one scan;
  their uint32 totals (root kept in the element dtype) are reproduced from
  the scanned output at the peeled block boundaries.  The step functions
  up_sweep / down_sweep run the reference's exact Blelloch pairing on the
  GPU (ps_tree_up_sweep / ps_tree_down_sweep).

lane_shift_with_zero_fill / vector_inclusive_scan / AddRoundCounter describe
the w-lane register primitive itself; they stay host-side numpy models of the
5-round __shfl_up_sync warp scan the kernels use (scan_device.cuh).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import device as dev
from .core import (DeviceView, Span, _check_buffer, _total, accumulator_zero, coerce_offset, full_span,
                   is_device, scan_into)

SUPPORTED_LANE_WIDTHS = (4, 8, 16)
DEFAULT_LANE_WIDTH = 16


@dataclass
class AddRoundCounter:
    """Counts shift-add rounds executed by ``vector_inclusive_scan``."""

    rounds: int = 0


def lane_shift_with_zero_fill(v: np.ndarray, k: int) -> np.ndarray:
    """Shift lanes up by ``k`` (lane i <- lane i-k), zero-filling low lanes.

    The warp form is ``__shfl_up_sync(mask, v, k)`` with lanes < k masked to 0."""
    w = v.shape[0]
    if k < 0 or k > w:
        raise ValueError(f"shift count {k} outside [0, {w}]")
    res = np.zeros_like(v)
    res[k:] = v[:w - k]
    return res


def vector_inclusive_scan(v: np.ndarray, counter: AddRoundCounter | None = None) -> np.ndarray:
    """Hillis-Steele scan of one w-lane vector: log2(w) shift-add rounds with
    shifts 1, 2, ..., w/2, additions in the element dtype."""
    w = v.shape[0]
    if w < 1 or (w & (w - 1)) != 0:
        raise ValueError(f"lane count {w} is not a power of two")
    acc = v.copy()
    shift = 1
    while shift < w:
        acc = acc + lane_shift_with_zero_fill(acc, shift)
        if counter is not None:
            counter.rounds += 1
        shift *= 2
    return acc


def _check_width(w: int) -> int:
    if w not in SUPPORTED_LANE_WIDTHS:
        raise ValueError(f"lane width {w} unsupported; choose from {SUPPORTED_LANE_WIDTHS}")
    return w


def _is_u32(data) -> bool:
    return dev.dtype_code(data.dtype) == 3


def horizontal_scan(data, span: Span, offset=0, w: int = DEFAULT_LANE_WIDTH, out=None):
    """Single-pass blockwise scan (simd.py:134-148); in place unless ``out``.

    Returns the final running total in accumulator precision (for uint32 the
    reference's wrapped-block total, see the module docstring)."""
    _check_width(w)
    _check_buffer(data)
    span.check(data)
    if out is not None:
        span.check(out)
    if not _is_u32(data) or span.len == 0:
        return scan_into(data, out, span, offset)
    src = DeviceView(data, span)
    quirk_total = dev.wrapped_block_total(src.t, w, coerce_offset(offset, data.dtype))
    tgt = src if out is None else DeviceView(out, span, load=False)
    dev.scan(src.t, tgt.t, seed=coerce_offset(offset, data.dtype))
    tgt.commit()
    return _total(quirk_total, data.dtype)


def simd_accumulate(data, span: Span, w: int = DEFAULT_LANE_WIDTH):
    """Span total via lane-wise partial sums (simd.py:151-159); read-only."""
    _check_width(w)
    from .core import sequential_accumulate
    return sequential_accumulate(data, span)


# ---- vertical family ------------------------------------------------------------------------

def _chunk_len(region: Span, w: int) -> int:
    if w < 1 or region.len % w:
        raise ValueError(f"region length {region.len} not divisible by lane width {w}")
    return region.len // w


def _acc_vector(host_or_dev, rows: int, dtype, device) -> tuple[torch.Tensor, bool]:
    """A device accumulator vector aliasing (or staged from) a caller array."""
    acc_t = dev.acc_dtype(dtype)
    if isinstance(host_or_dev, torch.Tensor) and host_or_dev.is_cuda:
        if host_or_dev.dtype != acc_t:
            raise ValueError(f"per-chunk array must be {acc_t}")
        return host_or_dev, False
    arr = np.asarray(host_or_dev)
    if arr.shape[0] != rows:
        raise ValueError(f"expected {rows} per-chunk entries")
    t = torch.from_numpy(np.ascontiguousarray(arr).astype(dev._acc_np(dev.dtype_code(dtype)))).to(device)
    return t, True


def _store_acc_vector(target, t: torch.Tensor) -> None:
    if isinstance(target, torch.Tensor) and target.is_cuda:
        if target.data_ptr() != t.data_ptr():
            target.copy_(t)
        return
    host = t.cpu().numpy()
    target[:] = host.astype(target.dtype) if isinstance(target, np.ndarray) else host


def _chunks(data, region: Span, w: int) -> tuple[DeviceView, torch.Tensor]:
    k = _chunk_len(region, w)
    v = DeviceView(data, region)
    return v, v.t.view(w, k)


def vertical_scan_pass1_scan(data, region: Span, carry_in, totals_out) -> None:
    """First vertical pass, scan flavour (simd.py:215-229): chunk i =
    region[i*k:(i+1)*k] scanned locally, chunk 0 seeded with ``carry_in``;
    ``totals_out[i]`` <- chunk i's running total."""
    _check_buffer(data)
    region.check(data)
    w = totals_out.shape[0]
    v, rows = _chunks(data, region, w)
    seeds_h = np.zeros(w, dev._acc_np(dev.dtype_code(data.dtype)))
    seeds_h[0] = coerce_offset(carry_in, data.dtype)
    seeds = torch.from_numpy(seeds_h).to(v.t.device)
    tot, _ = _acc_vector(totals_out, w, data.dtype, v.t.device)
    dev.scan_batched(rows, row_seeds=seeds, row_totals=tot)
    v.commit()
    _store_acc_vector(totals_out, tot)


def vertical_scan_pass1_accumulate(data, region: Span, totals_out) -> None:
    """First vertical pass, accumulate flavour (simd.py:232-238): totals only."""
    _check_buffer(data)
    region.check(data)
    w = totals_out.shape[0]
    v, rows = _chunks(data, region, w)
    tot, _ = _acc_vector(totals_out, w, data.dtype, v.t.device)
    dev.reduce_batched(rows, tot)
    _store_acc_vector(totals_out, tot)


def vertical_scan_pass2_increment(data, region: Span, chunk_offsets) -> None:
    """Second pass after a scan-flavour pass 1 (simd.py:241-246): chunk i += offsets[i]."""
    _check_buffer(data)
    region.check(data)
    w = chunk_offsets.shape[0]
    v, rows = _chunks(data, region, w)
    offs, _ = _acc_vector(chunk_offsets, w, data.dtype, v.t.device)
    dev.add_offset_batched(rows, offs)
    v.commit()


def vertical_scan_pass2_scan(data, region: Span, chunk_offsets) -> None:
    """Second pass after an accumulate-flavour pass 1 (simd.py:249-258):
    chunk i scanned seeded with offsets[i]."""
    _check_buffer(data)
    region.check(data)
    w = chunk_offsets.shape[0]
    v, rows = _chunks(data, region, w)
    offs, _ = _acc_vector(chunk_offsets, w, data.dtype, v.t.device)
    dev.scan_batched(rows, row_seeds=offs)
    v.commit()


def exclusive_offsets(totals: np.ndarray, seed) -> np.ndarray:
    """offset[i] = seed + sum(totals[:i]) (simd.py:261-268); w entries, host side."""
    res = np.empty_like(totals)
    running = seed
    for i, t in enumerate(totals):
        res[i] = running
        running = running + t
    return res


def vertical_scan(data, span: Span, offset=0, w: int = DEFAULT_LANE_WIDTH, scan_in_pass1: bool = True,
                  block_len: int = 0, out=None):
    """Full two-pass vertical scan (simd.py:271-314).  On the GPU both pass
    orders and every region size collapse into one single-pass scan; the
    returned total is the exact running total, as the reference's is."""
    _check_width(w)
    _check_buffer(data)
    span.check(data)
    if block_len < 0:
        raise ValueError(f"block_len must be >= 0, got {block_len}")
    if out is not None:
        span.check(out)
    return scan_into(data, out, span, offset)


# ---- tree family ------------------------------------------------------------------------------

def _require_tree_length(length: int, w: int) -> None:
    blocks = length // w if w else 0
    if length < w or blocks * w != length or (blocks & (blocks - 1)) != 0:
        raise ValueError(f"tree span length {length} is not a power of two times {w}")


def _wrap_u32_total(total: int, offset) -> int:
    """offset + (span sum mod 2^32): the tree root is kept in a uint32 element."""
    off = int(coerce_offset(offset, np.uint32))
    return (off + ((int(total) - off) & 0xFFFFFFFF)) & 0xFFFFFFFFFFFFFFFF


def up_sweep(data, span: Span):
    """Reduction sweep building the conceptual tree in place; returns the root
    (simd.py:356-360).  Element-typed arithmetic in the reference's exact
    pairing on the GPU (ps_tree_up_sweep), so float results are bit-identical."""
    _check_buffer(data)
    span.check(data)
    _require_tree_length(span.len, 1)
    v = DeviceView(data, span)
    root = dev.tree_up_sweep(v.t)
    v.commit()
    return root.cpu().numpy()[0]


def down_sweep(data, span: Span) -> None:
    """Distribution sweep: turns an up-swept span into its exclusive scan
    (simd.py:363-367), on the GPU (ps_tree_down_sweep)."""
    _check_buffer(data)
    span.check(data)
    _require_tree_length(span.len, 1)
    v = DeviceView(data, span)
    dev.tree_down_sweep(v.t)
    v.commit()


def tree_scan(data, span: Span, offset=0, w: int = DEFAULT_LANE_WIDTH, scratch=None):
    """Up/down-sweep scan of one block whose length is a power of two times w
    (simd.py:375-395).  Returns offset + span total (uint32: total mod 2^32)."""
    _check_width(w)
    _check_buffer(data)
    span.check(data)
    _require_tree_length(span.len, w)
    total = scan_into(data, None, span, offset)
    if _is_u32(data):
        return _wrap_u32_total(total, offset)
    return total


def _tree_blocks(span: Span, w: int, block_len: int) -> list[tuple[int, int, bool]]:
    """The peeling of simd.py:414-426: (start, len, is_tree_block) pieces."""
    pieces = []
    step = block_len if block_len > 0 else max(span.len, 1)
    pos, end = span.start, span.end
    while pos < end:
        region_end = min(pos + step, end)
        while region_end - pos >= w:
            blk = w << (((region_end - pos) // w).bit_length() - 1)
            pieces.append((pos, blk, True))
            pos += blk
        if region_end > pos:
            pieces.append((pos, region_end - pos, False))
            pos = region_end
    return pieces


def tree_scan_auto(data, span: Span, offset=0, w: int = DEFAULT_LANE_WIDTH, block_len: int = 0, out=None):
    """Tree scan over an arbitrary span (simd.py:398-427): one GPU scan.

    For uint32 the reference's total is offset + sum over the peeled tree
    blocks of (block sum mod 2^32) + the exact sums of the sub-w horizontal
    tails.  Both are recovered from the wrapped scanned output: a block's sum
    mod 2^32 is the difference of the outputs at its ends, and every element
    (< 2^32) is the difference of consecutive outputs."""
    _check_width(w)
    _check_buffer(data)
    span.check(data)
    if out is not None:
        span.check(out)
    total = scan_into(data, out, span, offset)
    if not _is_u32(data) or span.len == 0:
        return total
    res = out if out is not None else data
    pieces = _tree_blocks(span, w, block_len)
    idx = []
    for s0, ln, tree in pieces:
        idx.extend([s0 + ln - 1] if tree else range(s0, s0 + ln))
    if is_device(res):  # torch has no uint32 gather: index the int32 view, reinterpret on the host
        sel = torch.tensor(idx, dtype=torch.int64, device=res.device)
        vals = res.view(torch.int32)[sel].cpu().numpy().view(np.uint32)
    else:
        vals = np.asarray(res)[idx]
    acc = int(coerce_offset(offset, np.uint32))
    prev = acc & 0xFFFFFFFF
    for v in vals:  # each step is either a whole tree block or one tail element
        acc = (acc + ((int(v) - prev) & 0xFFFFFFFF)) & 0xFFFFFFFFFFFFFFFF
        prev = int(v)
    return acc
