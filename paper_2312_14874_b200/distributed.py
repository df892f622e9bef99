"""Multi-GPU sharded scan: one process per GPU, contiguous shards.

This is the paper's partition-then-two-pass structure (engine.py:278-344,
plan.py:160-178) mapped onto the GPUs of one box:

  * partition: the EQUAL layout -- rank g owns span g of ``equal_shards`` (the
    reference's compute_layout EQUAL split, aligned to the 32-byte vector);
  * pass 1 / ledger / barrier: each rank produces one 8-byte shard total and
    the G totals are exchanged with one all-gather (NCCL over NVLink/NVSwitch
    under torchrun) -- the ledger fold ``offset = base + sum(row[:j])``
    (engine.py:329-331) becomes ``carry_g = seed + sum(totals[:g])``,
    evaluated *on the device* by the consuming kernel (seed_terms), so no
    host round trip sits between the passes;
  * pass 2: a carry-in look-back scan.

Two schemes, named as in plan.py:24-37:
  ACCUMULATE_SCAN_EQUAL  reduce-then-scan: read n/G, exchange, read+write n/G
                         (3n/G bytes per GPU; the last rank's reduce is still
                         needed for the global total)
  SCAN_INCREMENT_EQUAL   scan-then-fixup: read+write n/G, exchange,
                         read+write n/G (4n/G bytes; rank 0 skips the fixup,
                         the paper's idle thread 0)

The local operations are injectable (``ops``) so the exchange logic is
testable on CPU processes with the gloo backend; the default -- and the only
product path -- is the CUDA library.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import device as dev
from .plan import SchemeId, equal_shards


class CudaOps:
    """The product's local ops: the sm_100a kernels (device.py)."""

    @staticmethod
    def reduce(x, seed=0):
        return dev.reduce(x, seed=seed)

    @staticmethod
    def scan(x, out, exclusive=False, seed=0, seed_terms=None):
        return dev.scan(x, out, exclusive=exclusive, seed=seed, seed_terms=seed_terms)

    @staticmethod
    def add_offset(x, delta=0, delta_terms=None):
        dev.add_offset(x, delta, delta_terms)


def shard_span(n: int, world: int, rank: int, elem_bytes: int = 8):
    """This rank's [start, start+len) of a length-n array (EQUAL layout,
    plan.py:160-166, non-final spans aligned to the 32-byte vector)."""
    return equal_shards(n, world, align=max(1, 32 // elem_bytes))[rank]


@dataclass
class ShardedScanResult:
    total: torch.Tensor         # global total (seed + everything), accumulator dtype
    shard_totals: torch.Tensor  # the G exchanged shard totals


class ShardedScan:
    """Scan a globally contiguous array whose rank-g piece lives on rank g."""

    def __init__(self, group=None, scheme: SchemeId = SchemeId.ACCUMULATE_SCAN_EQUAL, ops=None):
        if scheme not in (SchemeId.ACCUMULATE_SCAN_EQUAL, SchemeId.SCAN_INCREMENT_EQUAL):
            raise ValueError("multi-GPU scans use the EQUAL schemes (reduce-then-scan or scan-then-fixup)")
        self.group = group
        self.scheme = scheme
        self.ops = ops if ops is not None else CudaOps()
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0

    def _exchange(self, local_total: torch.Tensor) -> torch.Tensor:
        """All-gather of one accumulator per rank (G x 8 bytes)."""
        if self.world == 1:
            return local_total.reshape(1)
        parts = [torch.empty_like(local_total) for _ in range(self.world)]
        dist.all_gather(parts, local_total, group=self.group)
        return torch.cat(parts)

    def __call__(self, shard: torch.Tensor, out: torch.Tensor | None = None, *, exclusive: bool = False,
                 seed=0, want_total: bool = True) -> ShardedScanResult:
        """Scan this rank's shard in the global order.  Returns the global
        total (device, accumulator dtype; None if ``want_total`` is False)
        and the exchanged shard totals.  Nothing is synchronised."""
        out = shard if out is None else out
        r = self.rank
        if self.scheme is SchemeId.ACCUMULATE_SCAN_EQUAL:
            totals = self._exchange(self.ops.reduce(shard))
            self.ops.scan(shard, out, exclusive=exclusive, seed=seed, seed_terms=totals[:r] if r else None)
            return ShardedScanResult(self.ops.reduce(totals, seed=seed) if want_total else None, totals)
        # scan-then-fixup: rank 0's local scan carries the seed, the others add
        # the sum of their predecessors' totals afterwards
        local = self.ops.scan(shard, out, exclusive=exclusive, seed=seed if r == 0 else 0)
        totals = self._exchange(local)
        if r:
            self.ops.add_offset(out, 0, totals[:r])
        return ShardedScanResult(self.ops.reduce(totals) if want_total else None, totals)
