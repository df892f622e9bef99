"""Fused shard-total exchange (ps_publish_total / ps_scan_mailbox, MailboxExchange)
emulated on ONE GPU: G virtual ranks with one mailbox each in local device memory,
launched in rank order so every wait is satisfied by an earlier launch (no kernel
ever waits on one that runs later -- the profiling guide's rule).  Across GPUs the
same addresses come from a symmetric-memory rendezvous and the stores travel over
NVLink; the protocol (slot layout, epoch parity, prev-epoch back-pressure, fixed
fold order, timeout) is what is tested here."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _exchanges(G):
    from paper_2312_14874_b200.distributed import MailboxExchange
    boxes = [torch.zeros(2 * G * 16, dtype=torch.uint8, device="cuda") for _ in range(G)]
    bases = [b.data_ptr() for b in boxes]
    return [MailboxExchange(boxes[g], bases, g) for g in range(G)]


def _data(dt, n, seed):
    r = np.random.default_rng(seed)
    if np.dtype(dt).kind == "f":
        return r.random(n, dtype=dt)
    return r.integers(0, 1001, n).astype(dt)


@pytest.mark.parametrize("G", [2, 3, 4])
@pytest.mark.parametrize("scheme", ["accumulate-scan", "scan-increment"])
@pytest.mark.parametrize("dt,n", [(np.int64, 3_000_017), (np.float32, 5_000_011), (np.int32, 40_001)])
def test_p2p_sharded_scan_emulated(G, scheme, dt, n):
    from paper_2312_14874_b200 import device as dev
    from paper_2312_14874_b200.distributed import ShardedScan, shard_span
    from paper_2312_14874_b200.plan import SchemeId
    ex = _exchanges(G)
    scans = [ShardedScan(scheme=SchemeId(scheme), exchange="p2p", mailbox=ex[g]) for g in range(G)]
    a = _data(dt, n, n + G)
    acc = np.float64 if np.dtype(dt).kind == "f" else np.int64
    for step, (seed, exclusive) in enumerate([(0, False), (5, True), (0, False), (7, False), (3, True)]):
        outs = []
        for g in range(G):  # rank order: every mailbox wait is satisfied by an earlier launch
            sp = shard_span(n, G, g, np.dtype(dt).itemsize)
            x = torch.from_numpy(a[sp.start:sp.end].copy()).cuda()
            o = torch.empty_like(x) if dt != np.int32 else torch.empty(x.shape, dtype=torch.int32, device="cuda")
            scans[g](x, o, exclusive=exclusive, seed=seed, want_total=False)
            outs.append(o)
        got = np.concatenate([o.cpu().numpy() for o in outs])
        inc = np.cumsum(a.astype(acc)) + seed
        want = np.concatenate([[seed], inc[:-1]]) if exclusive else inc
        if np.dtype(dt).kind == "f":
            assert np.max(np.abs(got - want) / np.maximum(np.abs(want), 1e-30)) <= 1e-6, step
        else:
            assert np.array_equal(got, want.astype(dt)), step
        # every rank can now fold the global total from its mailbox
        e = ex[0].epoch
        extra = seed if scheme == "accumulate-scan" else 0
        for g in range(G):
            t = dev.scan_mailbox(None, None, ex[g].slots(e), G, e, seed=extra, timeout=ex[g].timeout,
                                 dtype=torch.from_numpy(a[:1]).dtype)
            tv = t.cpu().item()
            if np.dtype(dt).kind == "f":
                assert abs(tv - inc[-1]) <= 1e-9 * inc[-1], (step, g)
            else:
                assert tv == int(inc[-1]), (step, g)
    for g in range(G):
        ex[g].check()


def test_p2p_timeout_does_not_hang():
    """A scan waiting for a total that is never published gives up after ~10 s
    and reports it, instead of hanging the GPU."""
    import time
    from paper_2312_14874_b200 import device as dev
    ex = _exchanges(2)
    x = torch.arange(1, 100_001, dtype=torch.int64, device="cuda")
    t0 = time.time()
    dev.scan_mailbox(x, None, ex[1].slots(1), 1, 1, timeout=ex[1].timeout)  # rank 0 never published
    torch.cuda.synchronize()
    assert 8 < time.time() - t0 < 60
    with pytest.raises(RuntimeError, match="timed out"):
        ex[1].check()


def test_p2p_under_stalls():
    """Stall injection in every role of the consuming kernels changes nothing."""
    from paper_2312_14874_b200 import device as dev
    from paper_2312_14874_b200.distributed import ShardedScan, shard_span
    from paper_2312_14874_b200.plan import SchemeId
    G, n = 3, 4_000_003
    ex = _exchanges(G)
    scans = [ShardedScan(scheme=SchemeId.ACCUMULATE_SCAN_EQUAL, exchange="p2p", mailbox=ex[g]) for g in range(G)]
    a = _data(np.int64, n, 1)
    with dev.stall_injection(seed=5, prob=0.2, max_ns=20000):
        for _ in range(3):
            outs = []
            for g in range(G):
                sp = shard_span(n, G, g, 8)
                x = torch.from_numpy(a[sp.start:sp.end].copy()).cuda()
                scans[g](x, None, want_total=False)
                outs.append(x)
            assert np.array_equal(np.concatenate([o.cpu().numpy() for o in outs]), np.cumsum(a))
    for g in range(G):
        ex[g].check()


def test_mailbox_self_test_emulated():
    """The setup self-test (publish rank+1, fold all slots) on emulated ranks:
    run rank 0's publish, then rank 1's, then both folds."""
    from paper_2312_14874_b200 import device as dev
    ex = _exchanges(2)
    for g in range(2):
        e, prev = ex[g].next_epoch()
        ex[g].publish(torch.tensor([g + 1], dtype=torch.int64, device="cuda"), e, prev)
    for g in range(2):
        got = dev.scan_mailbox(None, None, ex[g].slots(1), 2, 1, timeout=ex[g].timeout, dtype=torch.int64)
        assert int(got.item()) == 3
        ex[g].check()
