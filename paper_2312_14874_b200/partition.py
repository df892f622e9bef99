"""Flag-driven compaction and partitioning on top of the exclusive offsets.

SURVEY.md §8(f)2: the paper motivates the prefix sum with exactly this use --
"determine the new offsets of data items during a partitioning step, where
prefix sums are computed from a previously constructed histogram or bitmap,
and then used as the new index values" (parallel filtering).
The reference package stops at the offsets (``sequential_inclusive_scan`` +
``exclusive_from_inclusive``, core.py:118-151); these functions add the
consumer:

* ``flagged_offsets(flags)``      exclusive int64 offsets + selected count
                                  (the cfg3 operation: one fused scan launch)
* ``select_flagged(values, flags)``    values whose flag is nonzero, in order
* ``partition_flagged(values, flags)`` stable partition: selected, then rejected

Each accepts CUDA tensors (results stay on the device) or numpy arrays (the
reference's calling convention: staged through the GPU, numpy returned).
``select_flagged`` / ``partition_flagged`` run ``ps_select``: tile counts ->
one-CTA offsets scan -> scatter through shared memory, order-preserving.
"""

from __future__ import annotations

import numpy as np
import torch

from . import device as dev


def _on_device(a):
    if isinstance(a, torch.Tensor):
        if not a.is_cuda:
            return a.cuda(), True
        return a, False
    if isinstance(a, np.ndarray):
        if a.ndim != 1:
            raise ValueError("expected a 1-D array")
        return torch.from_numpy(np.ascontiguousarray(a)).cuda(), True
    raise ValueError(f"expected a numpy array or torch tensor, got {type(a).__name__}")


def _back(t: torch.Tensor, like):
    if isinstance(like, np.ndarray):
        return t.cpu().numpy()
    if isinstance(like, torch.Tensor) and not like.is_cuda:
        return t.cpu()
    return t


def flagged_offsets(flags):
    """Exclusive prefix sum of 0/1 (or count) flags into int64 positions.

    Returns ``(offsets, total)``: ``offsets[i]`` = number of selected elements
    before i, ``total`` (Python int) = all selected -- the reference's
    ``exclusive_from_inclusive`` return value (core.py:141-151)."""
    f, staged = _on_device(flags)
    if f.dtype == torch.bool:
        f = f.to(torch.int32)
    if f.dtype not in (torch.int32, torch.int64, torch.uint32, torch.uint64):
        raise ValueError(f"flags must be an integer dtype, got {f.dtype}")
    wide = torch.int64 if f.dtype in (torch.int32, torch.int64) else torch.uint64
    out = torch.empty(f.shape, dtype=wide, device=f.device)
    if f.numel() == 0:
        return _back(out, flags), 0
    total = dev.scan(f, out, exclusive=True)
    return _back(out, flags), int(total.cpu().item())


def select_flagged(values, flags):
    """``values[flags != 0]`` in order (stream compaction)."""
    v, _ = _on_device(values)
    f, _ = _on_device(flags)
    out, count = dev.select(v, f)
    k = int(count.cpu().item())
    return _back(out[:k], values)


def partition_flagged(values, flags):
    """Stable partition: ``(concat(values[flags != 0], values[flags == 0]), k)``."""
    v, _ = _on_device(values)
    f, _ = _on_device(flags)
    out, count = dev.select(v, f, partition=True)
    return _back(out, values), int(count.cpu().item())
