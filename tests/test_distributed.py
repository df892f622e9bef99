"""Multi-process (gloo, CPU) tests of the sharded scan's host logic.

The product's local operations are CUDA kernels; here they are replaced by
the C oracle (test-only OracleOps) so the shard split, the all-gather of the
shard totals, the carry fold and both schemes (reduce-then-scan =
ACCUMULATE_SCAN_EQUAL, scan-then-fixup = SCAN_INCREMENT_EQUAL) run on CPU
processes exactly as they do one-process-per-GPU under torchrun + NCCL.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class OracleOps:
    """Local ops on CPU tensors through the C oracle (test infrastructure)."""

    def __init__(self):
        from oracle import oracle
        self.o = oracle

    @staticmethod
    def _acc(x):
        return torch.float64 if x.dtype.is_floating_point else torch.int64

    def reduce(self, x, seed=0):
        a = x.numpy()
        tot = self.o.accumulate(a, 0, a.shape[0]) + seed
        return torch.tensor([tot], dtype=self._acc(x))

    def scan(self, x, out, exclusive=False, seed=0, seed_terms=None):
        s = seed + (seed_terms.sum().item() if seed_terms is not None else 0)
        a = x.numpy().copy()
        tot = self.o.scan(a, 0, a.shape[0], s)
        if exclusive:
            res = np.concatenate([[s], a[:-1]]).astype(a.dtype) if a.shape[0] else a
        else:
            res = a
        out.copy_(torch.from_numpy(res))
        return torch.tensor([tot], dtype=self._acc(x))

    def add_offset(self, x, delta=0, delta_terms=None):
        d = delta + (delta_terms.sum().item() if delta_terms is not None else 0)
        a = x.numpy().copy()
        self.o.increment(a, 0, a.shape[0], d)
        x.copy_(torch.from_numpy(a))


CASES = [(d, excl, seed) for d in ("int64", "float32") for excl, seed in ((False, 0), (True, 7))]
N = 100_003


def _global_input(dtype_name):
    rng = np.random.default_rng(123)
    if dtype_name == "int64":
        return rng.integers(0, 1001, N, dtype=np.int64)
    return rng.random(N, dtype=np.float32)


def _worker(rank, world, port, scheme_name, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2312_14874_b200.distributed import ShardedScan, shard_span
        from paper_2312_14874_b200.plan import SchemeId

        results = []
        for dtype_name, exclusive, seed in CASES:
            g = _global_input(dtype_name)
            sp = shard_span(N, world, rank, g.dtype.itemsize)
            shard = torch.from_numpy(g[sp.start:sp.end].copy())
            out = torch.empty_like(shard)
            res = ShardedScan(scheme=SchemeId(scheme_name), ops=OracleOps())(shard, out, exclusive=exclusive,
                                                                            seed=seed)
            results.append((sp.start, sp.len, out.numpy(), res.total.item()))
        parts = [None] * world
        dist.all_gather_object(parts, results)
        if rank == 0:
            q.put(parts)
    finally:
        dist.destroy_process_group()


def _run(world, scheme_name):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, scheme_name, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return parts


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("scheme", ["accumulate-scan", "scan-increment"])
def test_sharded_scan_matches_global_scan(world, scheme):
    parts = _run(world, scheme)
    for ci, (dtype_name, exclusive, seed) in enumerate(CASES):
        g = _global_input(dtype_name)
        inc = np.cumsum(g.astype(np.float64 if dtype_name == "float32" else np.int64)) + seed
        want = np.concatenate([[seed], inc[:-1]]) if exclusive else inc
        mine = sorted((p[ci] for p in parts), key=lambda r: r[0])
        got = np.concatenate([r[2] for r in mine])
        assert sum(r[1] for r in mine) == N  # exact cover
        ctx = f"{world} ranks {scheme} {dtype_name} excl={exclusive}"
        if dtype_name == "int64":
            assert np.array_equal(got, want.astype(np.int64)), ctx
            assert all(int(r[3]) == int(inc[-1]) for r in mine), ctx
        else:
            rel = np.abs(got.astype(np.float64) - want) / np.maximum(np.abs(want), 1e-30)
            assert rel.max() <= 1e-6, ctx
            assert all(abs(r[3] - inc[-1]) <= 1e-9 * inc[-1] for r in mine), ctx


def test_shard_span_exact_cover_and_alignment():
    from paper_2312_14874_b200.distributed import shard_span
    for n in (0, 1, 7, 100, 4096, 10**6 + 3):
        for world in (1, 2, 3, 8):
            spans = [shard_span(n, world, r, 8) for r in range(world)]
            assert sum(s.len for s in spans) == n
            pos = 0
            for s in spans:
                assert s.start == pos
                pos += s.len
            if n >= world * 4:
                for s in spans[:-1]:
                    assert s.len % 4 == 0  # 32-byte vector alignment for int64


def test_sharded_scan_rejects_plus_one_schemes():
    from paper_2312_14874_b200.distributed import ShardedScan
    from paper_2312_14874_b200.plan import SchemeId
    with pytest.raises(ValueError):
        ShardedScan(scheme=SchemeId.ACCUMULATE_SCAN_PLUS_ONE)


# ---- engine-compatible multi-GPU executor (DistributedScanEngine) -----------------------

class FailingOps(OracleOps):
    """OracleOps whose scan raises on one rank (worker-failure propagation)."""

    def __init__(self, fail_rank):
        super().__init__()
        self.fail_rank = fail_rank

    def scan(self, x, out, exclusive=False, seed=0, seed_terms=None):
        if dist.get_rank() == self.fail_rank:
            raise OSError("injected device failure")
        return super().scan(x, out, exclusive, seed, seed_terms)


def _engine_worker(rank, world, port, q):
    import random
    import time

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2312_14874_b200.distributed import DistributedScanEngine, shard_span
        from paper_2312_14874_b200.engine import ScanRequest
        from paper_2312_14874_b200.plan import Role, SchemeId

        eng = DistributedScanEngine(ops=OracleOps())
        rng = random.Random(100 + rank)
        calls = []

        def delay(worker, iteration, phase):
            calls.append((worker, iteration, phase))
            if rng.random() < 0.5:
                time.sleep(rng.random() * 2e-3)

        g = _global_input("int64")
        sp = shard_span(N, world, rank, 8)
        res = []
        for scheme in SchemeId:
            shard = torch.from_numpy(g[sp.start:sp.end].copy())
            out = torch.empty_like(shard)
            total = eng.run(ScanRequest(data=shard, out=out, scheme=scheme, collect_stats=True, delay_hook=delay))
            st = eng.last_stats
            p1, p2 = st.roles[0]
            res.append((scheme.name, sp.start, out.numpy(), int(total), st.iterations, st.kernel_launches,
                        st.bytes_moved, [(t, role.value, ln) for t, role, ln in p1],
                        [(t, role.value, ln) for t, role, ln in p2]))
        # failure on rank 1 -> RuntimeError on every rank, nobody hangs
        errs = []
        shard = torch.from_numpy(g[sp.start:sp.end].copy())
        try:
            DistributedScanEngine(ops=FailingOps(1)).run(ScanRequest(data=shard, scheme=SchemeId.SCAN_INCREMENT_EQUAL))
        except RuntimeError as exc:
            errs.append((str(exc), type(exc.__cause__).__name__ if exc.__cause__ else None))
        parts = [None] * world
        dist.all_gather_object(parts, (res, calls, errs))
        if rank == 0:
            q.put(parts)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_engine_schemes_stats_hooks_failures(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_engine_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = _global_input("int64")
    want = np.cumsum(g)
    from paper_2312_14874_b200.plan import SchemeId
    for si, scheme in enumerate(SchemeId):
        rows = sorted((parts[r][0][si] for r in range(world)), key=lambda x: x[1])
        got = np.concatenate([x[2] for x in rows])
        assert np.array_equal(got, want), scheme
        assert all(x[3] == int(want[-1]) for x in rows), scheme
        for rank, x in enumerate(sorted(rows, key=lambda x: x[1])):
            assert x[4] == 1
            p1, p2 = x[7], x[8]
            assert [t for t, _, _ in p1] == list(range(world))
            assert sum(ln for _, _, ln in p1) == N
            if "ACCUMULATE" in scheme.name:
                assert {role for _, role, _ in p1} == {"accumulate"} and {role for _, role, _ in p2} == {"scan"}
                assert x[6] == 3 * 8 * (x[2].shape[0])
            else:
                assert {role for _, role, _ in p2} == {"increment"} and [t for t, _, _ in p2] == list(range(1, world))
    for r in range(world):
        calls = parts[r][1]
        assert calls == [(r, 0, ph) for _ in SchemeId for ph in ("pass1", "pass2")]
        errs = parts[r][2]
        assert len(errs) == 1
        if r == 1:
            assert errs[0] == ("rank 1 failed", "OSError")
        else:
            assert errs[0][0] == "a peer rank failed"


def test_distributed_engine_single_process_and_validation():
    from paper_2312_14874_b200.distributed import DistributedScanEngine
    from paper_2312_14874_b200.engine import ScanRequest
    eng = DistributedScanEngine(ops=OracleOps())
    x = torch.arange(1, 11, dtype=torch.int64)
    assert eng.run(ScanRequest(data=x)) == 55
    assert x.tolist() == list(np.cumsum(np.arange(1, 11)))
    with pytest.raises(ValueError):
        eng.run(ScanRequest(data=x, scheme="bogus"))


def test_sharded_scan_exchange_validation_and_single_rank():
    from paper_2312_14874_b200.distributed import ShardedScan
    with pytest.raises(ValueError):
        ShardedScan(exchange="carrier-pigeon")
    s = ShardedScan(exchange="p2p", ops=OracleOps())  # one process: nothing to exchange
    assert s.mailbox is None
    x = torch.arange(1, 6, dtype=torch.int64)
    out = torch.empty_like(x)
    res = s(x, out)
    assert out.tolist() == [1, 3, 6, 10, 15] and int(res.total.item()) == 15


def test_bench_falls_back_to_nccl_when_p2p_is_unavailable():
    import bench
    from paper_2312_14874_b200.plan import SchemeId

    class Fake:
        def __init__(self, scheme, exchange):
            if exchange == "p2p":
                raise RuntimeError("no symmetric memory here")
            self.exchange = exchange

    obj, label = bench.make_sharded(SchemeId.ACCUMULATE_SCAN_EQUAL, "p2p", 4, cls=Fake)
    assert obj.exchange == "nccl" and label.startswith("nccl (p2p unavailable")
    obj, label = bench.make_sharded(SchemeId.ACCUMULATE_SCAN_EQUAL, "nccl", 4, cls=Fake)
    assert label == "nccl"
