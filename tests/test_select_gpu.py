"""Stream compaction / stable partition (ps_select, partition.py) against
numpy boolean masking -- bit-exact (values are moved, never combined)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

SIZES = [1, 7, 255, 8191, 8192, 8193, 3 * 8192 + 17, 100_003, (1 << 20) + 13]
VALUE_DTYPES = [np.int32, np.float32, np.int64, np.float64, np.uint32, np.uint64]
FLAG_DTYPES = [np.bool_, np.uint8, np.int32, np.uint32, np.int64, np.float32]


def _values(n, dt, seed):
    r = np.random.default_rng(seed)
    if np.dtype(dt).kind == "f":
        return r.standard_normal(n).astype(dt)
    info = np.iinfo(dt)
    return r.integers(info.min, info.max, n, dtype=dt, endpoint=True)


def _flags(n, dt, p, seed):
    r = np.random.default_rng(seed + 1)
    sel = r.random(n) < p
    if dt == np.bool_:
        return sel
    f = np.zeros(n, dt)
    # selected flags carry assorted nonzero patterns, not just 1
    nz = r.integers(1, 100, n).astype(dt)
    f[sel] = nz[sel]
    return f


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _expect(v, f, partition):
    sel = f != 0
    if partition:
        return np.concatenate([v[sel], v[~sel]]), int(sel.sum())
    return v[sel], int(sel.sum())


@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("partition", [False, True])
def test_select_sizes(n, partition):
    from paper_2312_14874_b200 import device as dev
    v = _values(n, np.int32, n)
    f = _flags(n, np.int32, 0.5, n)
    out, count = dev.select(_dev(v), _dev(f), partition=partition)
    want, k = _expect(v, f, partition)
    assert int(count.item()) == k
    got = out.cpu().numpy()
    assert np.array_equal(got[:len(want)], want)


@pytest.mark.parametrize("vdt", VALUE_DTYPES)
@pytest.mark.parametrize("fdt", FLAG_DTYPES)
def test_select_dtypes(vdt, fdt):
    from paper_2312_14874_b200 import device as dev
    n = 5 * 8192 + 333
    v = _values(n, vdt, 3)
    f = _flags(n, fdt, 0.3, 3)
    for partition in (False, True):
        out, count = dev.select(_dev(v), _dev(f), partition=partition)
        want, k = _expect(v, f, partition)
        assert int(count.item()) == k
        assert np.array_equal(out.cpu().numpy()[:len(want)].view(np.uint8), want.view(np.uint8))


@pytest.mark.parametrize("p", [0.0, 0.001, 0.5, 0.999, 1.0])
def test_select_densities(p):
    from paper_2312_14874_b200 import partition as part
    n = 200_000
    v = _values(n, np.int64, 9)
    f = _flags(n, np.uint8, p, 9)
    got = part.select_flagged(v, f)
    assert np.array_equal(got, v[f != 0])
    pg, k = part.partition_flagged(v, f)
    assert k == int((f != 0).sum())
    assert np.array_equal(pg, np.concatenate([v[f != 0], v[f == 0]]))


@pytest.mark.parametrize("shift_v,shift_f", [(1, 0), (0, 3), (5, 5), (2, 7)])
def test_select_misaligned_views(shift_v, shift_f):
    """Buffers that are not 32-byte aligned take the element-wise path."""
    from paper_2312_14874_b200 import device as dev
    n = 4 * 8192 + 9
    v = _values(n + 8, np.float32, 4)
    f = _flags(n + 8, np.int32, 0.4, 4)
    tv, tf = _dev(v), _dev(f)
    vv, ff = tv[shift_v:shift_v + n], tf[shift_f:shift_f + n]
    for partition in (False, True):
        out, count = dev.select(vv, ff, partition=partition)
        want, k = _expect(v[shift_v:shift_v + n], f[shift_f:shift_f + n], partition)
        assert int(count.item()) == k
        assert np.array_equal(out.cpu().numpy()[:len(want)], want)


def test_select_empty_and_errors():
    from paper_2312_14874_b200 import device as dev
    v = torch.empty(0, dtype=torch.int32, device="cuda")
    out, count = dev.select(v, torch.empty(0, dtype=torch.uint8, device="cuda"))
    assert int(count.item()) == 0
    x = torch.arange(10, dtype=torch.int32, device="cuda")
    with pytest.raises(ValueError):
        dev.select(x, torch.ones(9, dtype=torch.uint8, device="cuda"))
    with pytest.raises(ValueError):
        dev.select(x, torch.ones(10, dtype=torch.uint8, device="cuda"), out=x)  # overlaps the input
    with pytest.raises(ValueError):
        dev.select(x, torch.ones(10, dtype=torch.uint8, device="cuda"), out=torch.empty(4, dtype=torch.int32,
                                                                                        device="cuda"))


def test_flagged_offsets_cfg3_semantics():
    """Exclusive offsets of 0/1 int32 flags (cfg3) and the returned total."""
    from paper_2312_14874_b200 import partition as part
    f = np.random.default_rng(2).integers(0, 2, 1_000_003, dtype=np.int32)
    off, total = part.flagged_offsets(f)
    assert off.dtype == np.int64
    assert total == int(f.sum())
    want = np.concatenate([[0], np.cumsum(f, dtype=np.int64)[:-1]])
    assert np.array_equal(off, want)
    # the offsets are the scatter destinations select uses
    v = np.arange(f.size, dtype=np.int64)
    got = part.select_flagged(v, f)
    assert np.array_equal(got, v[f != 0])
    assert np.array_equal(off[f != 0], np.arange(total))


def test_select_full_size_cfg3_flags():
    """2^28 Bernoulli(0.5) int32 flags (the cfg3 input) selecting int32 values."""
    from paper_2312_14874_b200 import device as dev
    n = 1 << 28
    g = torch.Generator(device="cuda").manual_seed(5)
    f = torch.randint(0, 2, (n,), dtype=torch.int32, device="cuda", generator=g)
    v = torch.arange(n, dtype=torch.int32, device="cuda")
    out, count = dev.select(v, f)
    k = int(count.item())
    assert k == int(f.sum().item())
    # values are their own indices: the compacted prefix is strictly increasing and
    # every entry is a selected index
    sel = out[:k]
    assert bool((sel[1:] > sel[:-1]).all().item())
    assert bool((f[sel.long()] != 0).all().item())
    del out
    out, count = dev.select(v, f, partition=True)
    rej = out[k:]
    assert bool((rej[1:] > rej[:-1]).all().item())
    assert bool((f[rej.long()] == 0).all().item())


@pytest.fixture
def select_kernel():
    from paper_2312_14874_b200 import _lib
    lib = _lib.load()
    prev = lib.ps_get_tuning(b"select_kernel")

    def set_(k):
        assert lib.ps_set_tuning(b"select_kernel", k) == 0

    yield set_
    lib.ps_set_tuning(b"select_kernel", prev)


@pytest.mark.parametrize("n", [1, 4095, 4096, 4097, 148 * 4096 - 3, 148 * 4096 + 5, 3 * 148 * 4096 + 4099, 5_000_011])
def test_single_pass_select_sizes(select_kernel, n):
    from paper_2312_14874_b200 import device as dev
    select_kernel(2)
    v = _values(n, np.int32, n)
    f = _flags(n, np.int32, 0.5, n)
    out, count = dev.select(_dev(v), _dev(f))
    want = v[f != 0]
    assert int(count.item()) == want.size
    assert np.array_equal(out.cpu().numpy()[:want.size], want)


@pytest.mark.parametrize("vdt", [np.int32, np.float32, np.int64, np.float64])
@pytest.mark.parametrize("fdt", [np.bool_, np.int32, np.int64])
@pytest.mark.parametrize("p", [0.0, 0.3, 1.0])
def test_single_pass_select_dtypes(select_kernel, vdt, fdt, p):
    from paper_2312_14874_b200 import device as dev
    select_kernel(2)
    n = 2 * 148 * 4096 + 777
    v = _values(n, vdt, 5)
    f = _flags(n, fdt, p, 5)
    out, count = dev.select(_dev(v), _dev(f))
    want = v[f != 0]
    assert int(count.item()) == want.size
    assert np.array_equal(out.cpu().numpy()[:want.size].view(np.uint8), want.view(np.uint8))


def test_single_pass_matches_three_launch_and_repeats(select_kernel):
    """Both paths agree bit for bit, and repeated single-pass calls (fresh epochs on
    a scratch that also held tile counts) stay correct."""
    from paper_2312_14874_b200 import device as dev
    n = 6_000_001
    v = _dev(_values(n, np.float32, 8))
    f = _dev(_flags(n, np.uint8, 0.37, 8))
    select_kernel(1)
    a, ca = dev.select(v, f)
    a = a[:int(ca.item())].clone()
    select_kernel(2)
    for _ in range(4):
        b, cb = dev.select(v, f)
        assert int(cb.item()) == a.numel()
        assert torch.equal(b[:a.numel()], a)
        select_kernel(1)
        dev.select(v, f)  # leaves tile counts in the shared scratch
        select_kernel(2)


def test_single_pass_misaligned_falls_back(select_kernel):
    from paper_2312_14874_b200 import device as dev
    select_kernel(2)
    n = 1_000_000
    v = _values(n + 3, np.int32, 2)
    f = _flags(n + 3, np.int32, 0.5, 2)
    out, count = dev.select(_dev(v)[1:n + 1], _dev(f)[3:n + 3])  # 4-byte offsets: not 16-byte aligned
    want = v[1:n + 1][f[3:n + 3] != 0]
    assert int(count.item()) == want.size
    assert np.array_equal(out.cpu().numpy()[:want.size], want)
