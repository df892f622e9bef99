"""CSR-segmented scans (ps_scan_segmented) through both kernels -- the
shared-memory-region kernel (seg_stream.cuh, default for inputs >= 32 MiB)
and the look-back tiles (segmented.cuh) -- against a numpy reference, over
segment-length distributions, dtype pairs, exclusive mode, totals, unaligned
views and sizes that leave boundary portions, plus the full-size 2^28 int32 ->
int64 case with 2^20 segments.  Integers bit-exact; floats within 1e-6 of the
float64 reference (the kernels carry float64)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture
def seg_kernel():
    from paper_2312_14874_b200 import _lib
    lib = _lib.load()
    saved = lib.ps_get_tuning(b"seg_kernel")

    def pin(k):
        assert lib.ps_set_tuning(b"seg_kernel", k) == 0

    yield pin
    lib.ps_set_tuning(b"seg_kernel", saved)


def _seg_reference(x: np.ndarray, offs: np.ndarray, exclusive: bool, acc):
    """Per-segment scans and totals from one running sum in the accumulator type
    (long double for floats: the difference of two running sums must resolve a
    segment's first, possibly tiny, element to well below 1e-6 of itself)."""
    if np.dtype(acc).kind == "f":
        acc = np.longdouble
    c = np.cumsum(x.astype(acc), dtype=acc)
    lens = np.diff(offs)
    starts = np.repeat(offs[:-1], lens)
    zero = acc(0)
    before = np.where(starts > 0, c[np.maximum(starts - 1, 0)], zero)
    if exclusive:  # the running sum before each element, minus the segment's base: exactly 0 at heads
        c_before = np.concatenate([np.zeros(1, acc), c[:-1]]).astype(acc)
        out = c_before - before
    else:
        out = c - before
    ends = offs[1:] - 1
    seg_before = np.where(offs[:-1] > 0, c[np.maximum(offs[:-1] - 1, 0)], zero)
    tots = np.where(lens > 0, c[np.maximum(ends, 0)] - seg_before, zero)
    return out, tots


def _offsets(kind: str, n: int, r) -> np.ndarray:
    if kind == "uniform":
        cuts = np.sort(r.integers(0, n + 1, max(1, n // 3000)))
    elif kind == "geometric":
        cuts = np.cumsum(r.geometric(1 / 40, n // 20))
    elif kind == "empties":
        cuts = np.sort(np.concatenate([r.integers(0, n + 1, n // 500), np.repeat(r.integers(0, n + 1, 40), 100)]))
    elif kind == "ones":
        cuts = np.arange(1, n)
    elif kind == "long":
        cuts = np.array([n // 3, 2 * n // 3])
    elif kind == "leading_empties":
        cuts = np.concatenate([np.zeros(5, np.int64), np.sort(r.integers(0, n + 1, 100)), np.full(4, n)])
        return np.concatenate([[0], cuts, [n]]).astype(np.int64)
    else:
        raise ValueError(kind)
    cuts = cuts[(cuts > 0) & (cuts < n)]
    return np.concatenate([[0], cuts, [n]]).astype(np.int64)


PAIRS = [(np.int32, np.int64), (np.int64, np.int64), (np.float32, np.float32), (np.float64, np.float64),
         (np.uint32, np.uint32), (np.int32, np.int32)]
TORCH = {np.int32: torch.int32, np.int64: torch.int64, np.float32: torch.float32, np.float64: torch.float64,
         np.uint32: torch.uint32}
ACC = {np.int32: np.int64, np.int64: np.int64, np.float32: np.float64, np.float64: np.float64,
       np.uint32: np.uint64}


def _draw(dt, n, r):
    if np.dtype(dt).kind == "f":
        return r.random(n).astype(dt)
    return r.integers(0, 1000, n).astype(dt)


def _check(got, want, dt_out, ctx):
    if np.dtype(dt_out).kind == "f":
        w = want.astype(np.float64)
        err = np.abs(got.astype(np.float64) - w) / np.maximum(np.abs(w), 1e-30)
        assert err.max() <= 1e-6, (ctx, err.max())
    else:
        assert np.array_equal(got, want.astype(dt_out)), ctx


def _run(dt_in, dt_out, x, offs, exclusive, view):
    from paper_2312_14874_b200 import device
    n = x.shape[0] - 1 if view else x.shape[0]
    base = torch.from_numpy(x).cuda()
    xt = base[1:] if view else base
    out_full = torch.empty(n + 1, dtype=TORCH[dt_out], device="cuda")
    out = out_full[1:] if view else out_full[:n]
    nseg = offs.shape[0] - 1
    acc_t = {np.int64: torch.int64, np.uint64: torch.uint64, np.float64: torch.float64}[ACC[dt_in]]
    tots = torch.full((nseg,), 7, dtype=acc_t, device="cuda")
    device.scan_segmented(xt, torch.from_numpy(offs).cuda(), out, exclusive=exclusive, seg_totals=tots)
    return out.cpu().numpy(), tots.cpu().numpy()


@pytest.mark.parametrize("kernel", [1, 2])
@pytest.mark.parametrize("kind", ["uniform", "geometric", "empties", "ones", "long", "leading_empties"])
def test_segment_distributions(ps_lib, seg_kernel, kernel, kind):
    seg_kernel(kernel)
    r = np.random.default_rng(hash(kind) % 1000 + kernel)
    n = 2_500_003  # several regions of the region kernel plus a boundary portion
    offs = _offsets(kind, n, r)
    for dt_in, dt_out in PAIRS[:3]:
        x = _draw(dt_in, n + 1, r)
        for view in (False, True):
            xs = x[1:] if view else x[:n]
            for excl in (False, True):
                got, tots = _run(dt_in, dt_out, x if view else x[:n], offs, excl, view)
                want, want_t = _seg_reference(xs, offs, excl, ACC[dt_in])
                ctx = (kernel, kind, np.dtype(dt_in).name, view, excl)
                _check(got, want, dt_out, ctx)
                _check(tots, want_t, ACC[dt_in], ctx)


@pytest.mark.parametrize("kernel", [1, 2])
@pytest.mark.parametrize("pair", PAIRS, ids=lambda p: f"{np.dtype(p[0]).name}-{np.dtype(p[1]).name}")
def test_dtype_pairs(ps_lib, seg_kernel, kernel, pair):
    seg_kernel(kernel)
    dt_in, dt_out = pair
    r = np.random.default_rng(5)
    for n in (1, 77, 70_001, 1_300_017):
        offs = _offsets("geometric" if n > 100 else "long", n, r) if n > 2 else np.array([0, n], np.int64)
        x = _draw(dt_in, n, r)
        for excl in (False, True):
            got, tots = _run(dt_in, dt_out, x, offs, excl, False)
            want, want_t = _seg_reference(x, offs, excl, ACC[dt_in])
            _check(got, want, dt_out, (kernel, pair, n, excl))
            _check(tots, want_t, ACC[dt_in], (kernel, pair, n, excl))


def test_kernels_agree_bitwise_on_integers(ps_lib, seg_kernel):
    r = np.random.default_rng(8)
    n = 4_000_037
    offs = _offsets("geometric", n, r)
    x = r.integers(-500, 500, n).astype(np.int64)
    seg_kernel(1)
    a, ta = _run(np.int64, np.int64, x, offs, False, False)
    seg_kernel(2)
    b, tb = _run(np.int64, np.int64, x, offs, False, False)
    assert np.array_equal(a, b) and np.array_equal(ta, tb)


def test_region_kernel_is_deterministic_for_floats(ps_lib, seg_kernel):
    seg_kernel(2)
    r = np.random.default_rng(9)
    n = 3_000_001
    offs = _offsets("uniform", n, r)
    x = r.standard_normal(n).astype(np.float32)
    runs = [_run(np.float32, np.float32, x, offs, False, False) for _ in range(3)]
    assert all(np.array_equal(runs[0][0], o) and np.array_equal(runs[0][1], t) for o, t in runs[1:])


def test_full_size_int32_to_int64_one_million_segments(ps_lib):
    """The bench line's workload: 2^28 int32 -> int64, 2^20 segments (default kernel choice)."""
    r = np.random.default_rng(10)
    n, nseg = 1 << 28, 1 << 20
    offs = np.concatenate([[0], np.sort(r.integers(1, n, nseg - 1)), [n]]).astype(np.int64)
    x = r.integers(0, 256, n, dtype=np.int32)
    got, tots = _run(np.int32, np.int64, x, offs, False, False)
    want, want_t = _seg_reference(x, offs, False, np.int64)
    assert np.array_equal(got, want)
    assert np.array_equal(tots, want_t)


@pytest.mark.parametrize("din,dout,rows,cols", [
    (np.int32, np.int64, 1 << 17, 250),    # unaligned rows (1000 bytes)
    (np.int32, np.int64, 1 << 17, 256),    # aligned rows: the rows kernel's domain, below its crossover
    (np.int32, np.int32, 1 << 16, 501),
    (np.int64, np.int64, 1 << 16, 250),
    (np.float32, np.float32, 1 << 17, 250),
    (np.float64, np.float64, 1 << 16, 127),
    (np.int32, np.int64, 2049, 16383),     # long rows the rows kernel cannot stream (not a multiple of 16 bytes)
    (np.float32, np.float32, 1500, 20001),
    (np.int64, np.int64, 700, 30001),
])
@pytest.mark.parametrize("exclusive", [False, True])
def test_short_rows_of_a_large_batch_run_on_the_region_kernel(ps_lib, seg_kernel, din, dout, rows, cols, exclusive):
    """ps_scan_batched on contiguous rows without seeds, >= 32 MiB in all -- short rows, and
    rows of any length whose byte size is not a multiple of 16: one segmented scan of the flat
    array with computed offsets on the shared-memory-region kernel; results and row totals
    against numpy, and against the look-back route."""
    from paper_2312_14874_b200 import device
    r = np.random.default_rng(rows + cols)
    fl = np.dtype(din).kind == "f"
    acc = np.float64 if fl else np.int64
    xh = (r.integers(0, 1024, (rows, cols)) / 1024.0).astype(din) if fl else r.integers(-50, 200, (rows, cols)).astype(din)
    assert xh.nbytes >= 32 << 20
    inc = np.cumsum(xh.astype(acc), axis=1)
    want = ((inc - xh.astype(acc)) if exclusive else inc).astype(dout)
    x = torch.from_numpy(xh).cuda()
    res = []
    for k in (0, 1):
        seg_kernel(k)
        out = torch.zeros((rows, cols), dtype=getattr(torch, np.dtype(dout).name), device="cuda")
        tots = torch.zeros(rows, dtype=getattr(torch, np.dtype(acc).name), device="cuda")
        device.scan_batched(x, out, exclusive=exclusive, row_totals=tots)
        torch.cuda.synchronize()
        got, gt = out.cpu().numpy(), tots.cpu().numpy()
        assert np.array_equal(got, want), (k, din, rows, cols, exclusive)  # the 2^-10 float grid sums exactly
        assert np.array_equal(gt, inc[:, -1]), (k, din, rows, cols)
        res.append(got)
    assert np.array_equal(res[0], res[1])


@pytest.fixture(scope="module")
def ps_lib():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2312_14874_b200 import _lib
    return _lib.load()
