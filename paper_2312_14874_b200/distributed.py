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
  * pass 2: a carry-in scan (the same 1-D kernel, seeded on the device).

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


class MailboxExchange:
    """The fused exchange's plumbing: a mailbox of 2 x G 16-byte slots on
    every GPU and the device array of all G mailbox addresses, so that
    ``ps_publish_total`` stores straight into the peers' memory over NVLink /
    NVSwitch and ``ps_scan_mailbox`` polls its own mailbox from inside the
    scan kernel (SURVEY.md §8(e) option ii) -- no collective launch, no host
    synchronisation between the passes.

    ``bases`` are the mailbox base addresses indexed by rank: from a
    symmetric-memory rendezvous across processes (``from_group``), or any
    list of device addresses the caller provides (single-process emulation
    in the tests)."""

    def __init__(self, own: torch.Tensor, bases: list, rank: int, keepalive=None):
        self.own = own
        self.world = len(bases)
        self.rank = rank
        self.bases = torch.tensor(bases, dtype=torch.int64, device=own.device)
        self.timeout = torch.zeros(1, dtype=torch.int32, device=own.device)
        self.epoch = 0
        self._keep = keepalive

    @classmethod
    def from_group(cls, group=None, device=None):
        import torch.distributed._symmetric_memory as symm_mem

        world = dist.get_world_size(group)
        rank = dist.get_rank(group)
        device = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        buf = symm_mem.empty(2 * world * 16, dtype=torch.uint8, device=device)
        buf.zero_()
        torch.cuda.synchronize(device)
        hdl = symm_mem.rendezvous(buf, group if group is not None else dist.group.WORLD)
        bases = [int(p) for p in hdl.buffer_ptrs]
        dist.barrier(group)
        ex = cls(buf, bases, rank, keepalive=hdl)
        ex.self_test(group)
        return ex

    def self_test(self, group=None) -> None:
        """One exchange of known values (rank + 1) through the real protocol;
        raises unless every rank sees the exact sum, so a broken peer mapping
        is caught at setup (callers fall back to the NCCL all-gather)."""
        e, prev = self.next_epoch()
        mine = torch.tensor([self.rank + 1], dtype=torch.int64, device=self.own.device)
        self.publish(mine, e, prev)
        got = dev.scan_mailbox(None, None, self.slots(e), self.world, e, timeout=self.timeout, dtype=torch.int64)
        ok = int(got.item()) == self.world * (self.world + 1) // 2 and int(self.timeout.item()) == 0
        flag = torch.tensor([1 if ok else 0], dtype=torch.int64, device=self.own.device)
        if dist.is_initialized():
            dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
        if not int(flag.item()):
            raise RuntimeError("mailbox exchange self-test failed")

    def next_epoch(self) -> tuple[int, int]:
        prev = self.epoch
        self.epoch += 1
        if self.epoch > 0x3FFFFFFF:  # never wraps in practice (one per call)
            raise RuntimeError("mailbox epoch space exhausted")
        return self.epoch, prev

    def slots(self, epoch: int) -> int:
        return self.own.data_ptr() + (epoch & 1) * self.world * 16

    def publish(self, total: torch.Tensor, epoch: int, prev: int) -> None:
        dev.publish_total(total, self.bases, self.rank, epoch, prev, self.own, self.timeout)

    def check(self) -> None:
        """Raise if an in-kernel mailbox wait gave up (synchronises)."""
        if int(self.timeout.item()):
            raise RuntimeError("mailbox exchange timed out: a peer never published its shard total")


class ShardedScan:
    """Scan a globally contiguous array whose rank-g piece lives on rank g.

    ``exchange``: "nccl" -- one all-gather of the G shard totals between the
    passes; "p2p" -- the fused exchange over peer memory (MailboxExchange):
    the reduce's total is stored straight into every peer's mailbox and the
    consuming kernel waits for its predecessors' totals itself."""

    def __init__(self, group=None, scheme: SchemeId = SchemeId.ACCUMULATE_SCAN_EQUAL, ops=None,
                 exchange: str = "nccl", mailbox: MailboxExchange | None = None):
        if scheme not in (SchemeId.ACCUMULATE_SCAN_EQUAL, SchemeId.SCAN_INCREMENT_EQUAL):
            raise ValueError("multi-GPU scans use the EQUAL schemes (reduce-then-scan or scan-then-fixup)")
        if exchange not in ("nccl", "p2p"):
            raise ValueError(f"exchange must be 'nccl' or 'p2p', got {exchange!r}")
        self.group = group
        self.scheme = scheme
        self.ops = ops if ops is not None else CudaOps()
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.exchange = exchange
        self.mailbox = mailbox
        if exchange == "p2p" and mailbox is None:
            self.mailbox = MailboxExchange.from_group(group) if self.world > 1 else None

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
        if self.exchange == "p2p" and self.mailbox is not None:
            return self._call_p2p(shard, out, exclusive, seed, want_total)
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


    def _call_p2p(self, shard, out, exclusive, seed, want_total):
        mb = self.mailbox
        r, g = mb.rank, mb.world
        e, prev = mb.next_epoch()
        if self.scheme is SchemeId.ACCUMULATE_SCAN_EQUAL:
            mb.publish(dev.reduce(shard), e, prev)
            total = dev.scan_mailbox(shard, out, mb.slots(e), r, e, exclusive=exclusive, seed=seed,
                                     timeout=mb.timeout)
        else:
            local = dev.scan(shard, out, exclusive=exclusive, seed=seed if r == 0 else 0)
            mb.publish(local, e, prev)
            if r:
                delta = dev.scan_mailbox(None, None, mb.slots(e), r, e, timeout=mb.timeout, dtype=shard.dtype)
                dev.add_offset(out, 0, delta)
        if not want_total:
            return ShardedScanResult(None, None)
        # the global total: seed + every rank's published total (all G slots of epoch e)
        extra = seed if self.scheme is SchemeId.ACCUMULATE_SCAN_EQUAL else 0
        tot = dev.scan_mailbox(None, None, mb.slots(e), g, e, seed=extra, timeout=mb.timeout, dtype=shard.dtype)
        return ShardedScanResult(tot, None)


class DistributedScanEngine:
    """Engine-compatible multi-GPU executor (engine.py:131-260 vocabulary).

    ``run(ScanRequest)`` scans this rank's shard (``request.data``, the
    rank-g piece of a globally contiguous array, EQUAL layout) in the global
    order and returns the global total as a Python number -- the reference's
    ``ScanEngine.run`` contract, with the GPUs of the process group in place of
    the engine's worker threads:

    * ``request.scheme`` is the reference's ``SchemeId``: the EQUAL schemes run
      as themselves (reduce-then-scan / scan-then-fixup); the PLUS_ONE
      variants are accepted and run as their EQUAL counterpart (the extra
      dilated partition balances CPU threads around the idle thread 0;
      GPU shards are equal by construction);
    * ``request.delay_hook(rank, 0, "pass1" | "pass2")`` is called on the host
      before each pass (engine.py:285-314), so delay-injection stress written
      against the reference drives this engine unchanged;
    * ``request.collect_stats`` fills ``last_stats`` (``RunStats``): one
      iteration, one exchange, the per-rank roles of both passes, this rank's
      kernel launches and HBM bytes (3n/G or 4n/G);
    * a failure on any rank raises ``RuntimeError`` chained from the cause
      (engine.py:241-243); ``ValueError`` passes through.
    """

    _EQUAL = {
        SchemeId.ACCUMULATE_SCAN_EQUAL: SchemeId.ACCUMULATE_SCAN_EQUAL,
        SchemeId.ACCUMULATE_SCAN_PLUS_ONE: SchemeId.ACCUMULATE_SCAN_EQUAL,
        SchemeId.SCAN_INCREMENT_EQUAL: SchemeId.SCAN_INCREMENT_EQUAL,
        SchemeId.SCAN_INCREMENT_PLUS_ONE: SchemeId.SCAN_INCREMENT_EQUAL,
    }

    def __init__(self, group=None, ops=None):
        self.group = group
        self.ops = ops if ops is not None else CudaOps()
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.last_stats = None

    def _all_ok(self, ok: bool) -> bool:
        """Every rank learns whether any rank failed (the engine's job.failed);
        all ranks reach this point, failed or not, so nobody blocks in a
        collective a failed peer never enters (engine.py:313-315)."""
        if not dist.is_initialized() or self.world == 1:
            return ok
        flag = torch.tensor([1 if ok else 0], dtype=torch.int64)
        if dist.get_backend(self.group) == "nccl":
            flag = flag.cuda()
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=self.group)
        return bool(flag.item())

    def run(self, request) -> object:
        from .engine import RunStats
        from .plan import Role

        scheme = self._EQUAL.get(request.scheme)
        if scheme is None:
            raise ValueError(f"unknown scheme {request.scheme!r}")
        shard = request.data
        out = shard if request.out is None else request.out
        hook = request.delay_hook
        r, g = self.rank, self.world
        n = shard.shape[0]
        ss = ShardedScan(self.group, scheme, self.ops)

        def phase(fn):
            try:
                return fn(), None
            except BaseException as exc:  # noqa: BLE001 - re-raised below, chained
                return None, exc

        def pass1():
            if hook is not None:
                hook(r, 0, "pass1")
            if scheme is SchemeId.ACCUMULATE_SCAN_EQUAL:
                return self.ops.reduce(shard)
            return self.ops.scan(shard, out, exclusive=False, seed=0)

        local, err = phase(pass1)
        if not self._all_ok(err is None):
            raise RuntimeError(f"rank {r} failed" if err is not None else "a peer rank failed") from err
        totals = ss._exchange(local)

        def pass2():
            if hook is not None:
                hook(r, 0, "pass2")
            if scheme is SchemeId.ACCUMULATE_SCAN_EQUAL:
                self.ops.scan(shard, out, exclusive=False, seed=0, seed_terms=totals[:r] if r else None)
            elif r:
                self.ops.add_offset(out, 0, totals[:r])
            return self.ops.reduce(totals)

        total, err = phase(pass2)
        if not self._all_ok(err is None):
            raise RuntimeError(f"rank {r} failed" if err is not None else "a peer rank failed") from err
        if request.collect_stats:
            sizes = self._shard_lengths(n)
            esize = shard.element_size()
            if scheme is SchemeId.ACCUMULATE_SCAN_EQUAL:
                p1 = [(t, Role.ACCUMULATE, sizes[t]) for t in range(g)]
                p2 = [(t, Role.SCAN, sizes[t]) for t in range(g)]
                launches, nbytes = 3, 3 * n * esize
            else:
                p1 = [(t, Role.SCAN, sizes[t]) for t in range(g)]
                p2 = [(t, Role.INCREMENT, sizes[t]) for t in range(1, g)]
                launches = 3 if r else 2
                nbytes = (4 if r else 2) * n * esize
            # here the two passes and the exchange ARE what ran (one per rank)
            self.last_stats = RunStats(iterations=1, barrier_waits=1, sync_points=2, roles=[(p1, p2)],
                                       kernel_launches=launches, bytes_moved=nbytes, reference_plan_only=False)
        return total.cpu().item()

    def _shard_lengths(self, n_local: int) -> list:
        """Every rank's shard length (one small all-gather; stats only)."""
        if not dist.is_initialized() or self.world == 1:
            return [n_local]
        parts = [None] * self.world
        dist.all_gather_object(parts, n_local, group=self.group)
        return parts
