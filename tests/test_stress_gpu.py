"""Overlap-safety stress on the GPU: in-kernel stall injection at every role
hand-off (device.stall_injection) must never change a result -- the GPU form
of the reference's delay_hook stress (pkg/tests/test_engine.py "stalls must
never corrupt the double-buffered sums", test_acceptance.py criterion 4).

Integer results are compared bit-exactly with numpy; float32 results must be
bit-identical to the unstalled run (the ledger folds every region total in a
fixed order, so timing never changes a float sum)."""

import contextlib

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@contextlib.contextmanager
def tuning(**kv):
    from paper_2312_14874_b200 import _lib
    lib = _lib.load()
    saved = {k: lib.ps_get_tuning(k.encode()) for k in kv}
    for k, v in kv.items():
        _lib.check(lib.ps_set_tuning(k.encode(), v), "ps_set_tuning")
    try:
        yield
    finally:
        for k, v in saved.items():
            lib.ps_set_tuning(k.encode(), v)


def _scan(x, exclusive=False):
    from paper_2312_14874_b200 import device as dev
    out = torch.empty_like(x)
    total = dev.scan(x, out, exclusive=exclusive)
    return out.cpu().numpy(), total.cpu().numpy()[0]


KERNELS = {
    "rounds": dict(scan_kernel=2, round_bytes=1 << 20),  # ~1 MiB regions: hundreds of hand-offs
    "rounds_lead1": dict(scan_kernel=2, round_bytes=1 << 20, round_lead=1),
    "tiles": dict(scan_kernel=1),
    "stream": dict(scan_kernel=3),
}


@pytest.mark.parametrize("kernel", sorted(KERNELS))
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_int64_scan_under_stalls(kernel, seed):
    from paper_2312_14874_b200 import device as dev
    r = np.random.default_rng(seed)
    a = r.integers(-1000, 1001, 6_000_007, dtype=np.int64)
    x = torch.from_numpy(a).cuda()
    with tuning(**KERNELS[kernel]), dev.stall_injection(seed=seed, prob=0.15, max_ns=30000):
        got, total = _scan(x)
    assert np.array_equal(got, np.cumsum(a))
    assert total == a.sum()


@pytest.mark.parametrize("kernel", sorted(KERNELS))
def test_float32_bitwise_stable_under_stalls(kernel):
    from paper_2312_14874_b200 import device as dev
    a = np.random.default_rng(9).random(5_000_011, dtype=np.float32)
    x = torch.from_numpy(a).cuda()
    with tuning(**KERNELS[kernel]):
        base, btot = _scan(x)
        for seed in (4, 5):
            with dev.stall_injection(seed=seed, prob=0.2, max_ns=20000):
                got, tot = _scan(x)
            assert np.array_equal(got.view(np.uint32), base.view(np.uint32)), seed
            assert tot == btot
    want = np.cumsum(a.astype(np.float64))
    assert np.max(np.abs(base - want) / np.maximum(want, 1e-30)) <= 1e-6


@pytest.mark.parametrize("rows_kernel", [1, 2])
def test_batched_rows_under_stalls(rows_kernel):
    from paper_2312_14874_b200 import device as dev
    a = np.random.default_rng(7).integers(0, 256, (700, 50_000), dtype=np.int32)
    x = torch.from_numpy(a).cuda()
    out = torch.empty(a.shape, dtype=torch.int64, device="cuda")
    with tuning(rows_kernel=rows_kernel), dev.stall_injection(seed=11, prob=0.2, max_ns=20000):
        dev.scan_batched(x, out, exclusive=True)
    want = np.cumsum(a, axis=1, dtype=np.int64) - a
    assert np.array_equal(out.cpu().numpy(), want)


@pytest.mark.parametrize("cols,dynamic,multi", [(3000, 1, 1), (3000, 0, 1), (50_000, 1, 0), (20_000, 0, 0)])
def test_rows_kernel_tickets_and_short_rows_under_stalls(cols, dynamic, multi):
    """Row tickets (dynamic) and several short rows per buffer (multi) with the
    producer / scanner hand-offs stalled at random: results exact, and the ticket
    counters still return to zero (a second launch on the same scratch is exact)."""
    from paper_2312_14874_b200 import device as dev
    a = np.random.default_rng(17).integers(0, 256, (1500, cols), dtype=np.int32)
    x = torch.from_numpy(a).cuda()
    want = np.cumsum(a, axis=1, dtype=np.int64)
    with tuning(rows_kernel=2, rows_dynamic=dynamic, rows_multi=multi):
        for rep in range(2):
            out = torch.empty(a.shape, dtype=torch.int64, device="cuda")
            tots = torch.empty(a.shape[0], dtype=torch.int64, device="cuda")
            with dev.stall_injection(seed=21 + rep, prob=0.2, max_ns=20000):
                dev.scan_batched(x, out, row_totals=tots)
            assert np.array_equal(out.cpu().numpy(), want), rep
            assert np.array_equal(tots.cpu().numpy(), want[:, -1]), rep


def test_stall_injection_restores_and_validates():
    from paper_2312_14874_b200 import _lib, device as dev
    lib = _lib.load()
    before = [lib.ps_get_tuning(k) for k in (b"stall_seed", b"stall_prob", b"stall_ns")]
    with dev.stall_injection(seed=3, prob=0.5, max_ns=1000):
        assert lib.ps_get_tuning(b"stall_prob") == 512
        assert lib.ps_get_tuning(b"stall_ns") == 1000
    assert [lib.ps_get_tuning(k) for k in (b"stall_seed", b"stall_prob", b"stall_ns")] == before
    with pytest.raises(ValueError):
        dev.stall_injection(prob=1.5)
    assert lib.ps_set_tuning(b"stall_prob", 2000) == _lib.PS_ERR_ARG
