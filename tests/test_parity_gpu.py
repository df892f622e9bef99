"""GPU parity: the CUDA path (through the C-ABI) against the reference's own
outputs (golden vectors), the C oracle, and numpy, on the reference's entry
points and on BASELINE.json's configs.

Tolerances: integer dtypes are compared bit-exactly.  float32 outputs must be
within rtol 1e-6 of the reference (its own harness allows 1e-5,
bench.py:24; BASELINE.json allows 1e-4): the GPU carries float64 like the
reference but reassociates.  On the config generators (multiples of 2^-24,
partial sums < 2^29) float64 partial sums are exact, so cfg2 is asserted
bit-exact.
"""

import numpy as np
import pytest
import torch

import golden_cases as G
from conftest import assert_scan_matches, make_data

pytestmark = pytest.mark.gpu

FLOAT_RTOL = 1e-6


@pytest.fixture(scope="module")
def ps():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2312_14874_b200 as ps
    from paper_2312_14874_b200 import _lib
    _lib.load()
    return ps


def _cuda(a: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _host(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy()


def _beyond_2_53(case, inp):
    return inp.dtype.kind == "i" and inp.size and np.abs(inp.astype(np.float64)).sum() >= 2.0**53


def _assert_total(got, case):
    want = G.total_of(case)
    if want is None:
        return
    if isinstance(want, float) and case["dtype"] in ("float32", "float64"):
        # the reference's horizontal / tree totals fold float32 block sums (simd.py:84-94,
        # :330-334), so they sit ~1 float32 ulp from the float64 running total
        rel = 1e-12 if case["op"] in ("sequential_inclusive_scan", "sequential_accumulate", "engine") else 1e-6
        assert got == pytest.approx(want, rel=rel, abs=1e-12), (got, want)
    else:
        assert int(got) == int(want), (got, want)


def _assert_array(got, want, ctx):
    if want.dtype.kind == "f":
        assert_scan_matches(got, want, rtol=FLOAT_RTOL, context=ctx)
    else:
        assert np.array_equal(got, want), ctx


SCAN_CASES = [c for c, _, _ in G.cases() if c["op"] in (
    "sequential_inclusive_scan", "horizontal_scan", "vertical_scan", "tree_scan", "tree_scan_auto",
    "sequential_accumulate", "sequential_increment", "exclusive_from_inclusive", "engine")]


@pytest.mark.parametrize("case", SCAN_CASES, ids=[G.case_id(c) for c in SCAN_CASES])
@pytest.mark.parametrize("where", ["cuda", "numpy"])
def test_golden_through_dropin(ps, case, where):
    _, arrays = G.load()
    inp, want = arrays[case["in"]], arrays[case["out"]]
    if _beyond_2_53(case, inp):
        pytest.skip("reference float64 accumulator is lossy here; see test_int64_beyond_2_53_is_exact")
    data = _cuda(inp) if where == "cuda" else inp.copy()
    op = case["op"]
    total = None
    out = None
    if op == "sequential_inclusive_scan":
        total = ps.sequential_inclusive_scan(data, ps.Span(case["start"], case["len"]), case["offset"])
    elif op == "horizontal_scan":
        if case["out_of_place"]:
            out = torch.zeros_like(data) if where == "cuda" else np.zeros_like(inp)
        total = ps.horizontal_scan(data, ps.Span(case["start"], case["len"]), case["offset"], case["w"], out=out)
    elif op == "vertical_scan":
        total = ps.vertical_scan(data, ps.Span(case["start"], case["len"]), case["offset"], case["w"],
                                 case["scan_in_pass1"], case["block_len"])
    elif op == "tree_scan":
        total = ps.tree_scan(data, ps.Span(case["start"], case["len"]), case["offset"], case["w"])
    elif op == "tree_scan_auto":
        total = ps.tree_scan_auto(data, ps.Span(case["start"], case["len"]), case["offset"], case["w"],
                                  case["block_len"])
    elif op == "sequential_accumulate":
        total = ps.sequential_accumulate(data, ps.Span(case["start"], case["len"]))
    elif op == "sequential_increment":
        ps.sequential_increment(data, ps.Span(case["start"], case["len"]), case["offset"])
    elif op == "exclusive_from_inclusive":
        total = ps.exclusive_from_inclusive(data, case["identity"])
    elif op == "engine":
        out = torch.empty_like(data) if where == "cuda" else np.empty_like(inp)
        req = ps.ScanRequest(data=data, out=out, kernel=case["kernel"], scheme=ps.SchemeId(case["scheme"]),
                             block_len=case["block_len"], threads=case["threads"])
        total = ps.execute(req)
    res = out if out is not None else data
    got = _host(res) if where == "cuda" else res
    _assert_array(got, want, G.case_id(case))
    if op == "sequential_accumulate" or op == "sequential_increment":
        assert np.array_equal(_host(data) if where == "cuda" else data, want)  # read-only / in place
    if total is not None:
        _assert_total(total, case)


def test_int64_beyond_2_53_is_exact(ps):
    """Divergence pin: above 2^53 the reference's float64 accumulator rounds;
    the GPU keeps exact int64 (two's complement) arithmetic."""
    x = np.array([1, 2, 3, 2**60, 2**62], np.int64)
    t = _cuda(x)
    total = ps.sequential_inclusive_scan(t, ps.full_span(t))
    assert np.array_equal(_host(t), np.cumsum(x))
    assert total == int(np.sum(x))


def test_widen_exclusive_golden(ps):
    from paper_2312_14874_b200 import device
    (case, inp, want), = list(G.cases("widen_exclusive"))
    x = _cuda(inp)
    out = torch.empty(inp.shape[0], dtype=torch.int64, device="cuda")
    total = device.scan(x, out, exclusive=True)
    assert np.array_equal(_host(out), want)
    assert int(total.item()) == G.total_of(case) == int(inp.sum())


def test_rows_widen_golden(ps):
    from paper_2312_14874_b200 import device
    (case, inp, want), = list(G.cases("rows_widen_inclusive"))
    x = _cuda(inp)
    out = torch.empty(inp.shape, dtype=torch.int64, device="cuda")
    tot = torch.empty(inp.shape[0], dtype=torch.int64, device="cuda")
    device.scan_batched(x, out, row_totals=tot)
    assert np.array_equal(_host(out), want)
    assert np.array_equal(_host(tot), want[:, -1])


# ---- edge cases: sizes around tile boundaries, alignment, in/out of place ----------------------

TILE = {np.int64: 4096, np.int32: 8192, np.uint32: 8192, np.float32: 8192, np.float64: 4096, np.uint64: 4096}
GENS = {
    np.int64: lambda r, n: r.integers(-1000, 1001, n, dtype=np.int64),
    np.int32: lambda r, n: r.integers(-(2**31), 2**31, n, dtype=np.int32),
    np.uint32: lambda r, n: r.integers(0, 2**32, n, dtype=np.uint32),
    np.uint64: lambda r, n: r.integers(0, 2**63, n, dtype=np.uint64),
    np.float32: lambda r, n: r.random(n, dtype=np.float32),
    np.float64: lambda r, n: r.random(n),
}


def _expected(x, seed=0, exclusive=False, out_dtype=None):
    out_dtype = out_dtype or x.dtype
    if x.dtype.kind == "f":
        inc = np.cumsum(x.astype(np.float64)) + float(seed)
    elif x.dtype == np.uint32 or x.dtype == np.uint64:
        inc = np.cumsum(x.astype(np.uint64)) + np.uint64(seed)
    else:
        inc = np.cumsum(x.astype(np.int64)) + np.int64(seed)
    if exclusive:
        inc = np.concatenate([np.array([seed], inc.dtype), inc[:-1]]) if len(inc) else inc
    return inc.astype(out_dtype)


@pytest.mark.parametrize("dt", list(GENS))
def test_sizes_around_tiles(ps, dt):
    from paper_2312_14874_b200 import device
    r = np.random.default_rng(11)
    T = TILE[dt]
    for n in (0, 1, 2, 31, 32, 33, T - 1, T, T + 1, 2 * T - 1, 33 * T + 5, 70 * T + 3):
        x = GENS[dt](r, n)
        for exclusive in (False, True):
            t = _cuda(x)
            out = torch.empty_like(t)
            seed = 7 if dt != np.float32 else 0.5
            total = device.scan(t, out, exclusive=exclusive, seed=seed)
            ctx = f"{dt.__name__} n={n} excl={exclusive}"
            _assert_array(_host(out), _expected(x, seed, exclusive), ctx)
            tv = total.cpu().numpy()[0]
            exp_total = (_expected(x, seed, False, np.float64 if x.dtype.kind == "f" else None)[-1]
                         if n else seed)
            if x.dtype.kind == "f":
                assert abs(float(tv) - float(exp_total)) <= 1e-9 * max(1.0, abs(float(exp_total))), ctx
            elif dt in (np.uint32, np.uint64):
                assert int(tv) == (int(x.astype(np.uint64).sum(dtype=np.uint64)) + 7) % 2**64, ctx
            else:
                assert int(tv) == int(x.astype(np.int64).sum()) + 7, ctx


@pytest.mark.parametrize("dt", [np.int64, np.float32, np.uint32, np.int32])
def test_unaligned_starts(ps, dt):
    from paper_2312_14874_b200 import device
    r = np.random.default_rng(3)
    T = TILE[dt]
    base = GENS[dt](r, 5 * T + 100)
    for s_in in range(0, 9):
        for s_out in (s_in, (s_in + 1) % 9, 0):
            n = 3 * T + 17
            x = _cuda(base)
            o = torch.zeros(base.shape[0] + 16, dtype=x.dtype, device="cuda")
            xin, xout = x[s_in:s_in + n], o[s_out:s_out + n]
            device.scan(xin, xout)
            _assert_array(_host(xout), _expected(base[s_in:s_in + n]), f"{dt.__name__} in@{s_in} out@{s_out}")
            assert np.array_equal(_host(x), base)  # out of place leaves the input alone
            # in place on the unaligned view
            device.scan(xin)
            _assert_array(_host(x)[s_in:s_in + n], _expected(base[s_in:s_in + n]), f"inplace@{s_in}")
            assert np.array_equal(_host(x)[:s_in], base[:s_in])
            assert np.array_equal(_host(x)[s_in + n:], base[s_in + n:])


@pytest.fixture
def force_kernel():
    """Pin the scan kernel (1 look-back, 2 cache-partitioned rounds) and a small
    L2 region so modest inputs still span many regions; restore afterwards."""
    from paper_2312_14874_b200 import _lib
    lib = _lib.load()
    saved = {k: lib.ps_get_tuning(k.encode()) for k in ("scan_kernel", "round_bytes", "rounds_min_bytes")}

    def pin(kernel, round_bytes=1 << 20):
        assert lib.ps_set_tuning(b"scan_kernel", kernel) == 0
        assert lib.ps_set_tuning(b"round_bytes", round_bytes) == 0

    yield pin
    for k, v in saved.items():
        lib.ps_set_tuning(k.encode(), v)


@pytest.mark.parametrize("kernel", [1, 2, 3])
@pytest.mark.parametrize("dt", [np.int64, np.float32, np.uint32, np.int32, np.float64])
def test_both_scan_kernels(ps, force_kernel, kernel, dt):
    from paper_2312_14874_b200 import device
    force_kernel(kernel)
    r = np.random.default_rng(21)
    for n in (1, 1000, 65_536, 1_000_003, 5_000_011):
        x = GENS[dt](r, n + 9)
        for s_in in (0, 3):
            for exclusive in (False, True):
                xs = x[s_in:s_in + n]
                t = _cuda(x)[s_in:s_in + n]
                o = torch.empty(x.shape[0], dtype=t.dtype, device="cuda")[s_in:s_in + n]
                seed = 5 if x.dtype.kind != "f" else 0.25
                tot = device.scan(t, o, exclusive=exclusive, seed=seed)
                ctx = f"kernel={kernel} {dt.__name__} n={n} s={s_in} excl={exclusive}"
                _assert_array(_host(o), _expected(xs, seed, exclusive), ctx)
                tv = tot.cpu()
                if x.dtype.kind == "f":
                    assert abs(tv.item() - (xs.astype(np.float64).sum() + seed)) <= 1e-9 * n + 1e-9, ctx
                elif dt == np.uint32:
                    assert int(tv.view(torch.int64).item()) == int(xs.astype(np.uint64).sum()) + 5, ctx
                else:
                    assert int(tv.item()) == int(xs.astype(np.int64).sum()) + 5, ctx


@pytest.mark.parametrize("inflight", [0, 1, 2, 5])
def test_stream_kernel_inflight_limit(ps, force_kernel, inflight):
    """The producer's bound on outstanding region loads changes only timing."""
    from paper_2312_14874_b200 import _lib, device
    lib = _lib.load()
    prev = lib.ps_get_tuning(b"stream_inflight")
    force_kernel(3)
    assert lib.ps_set_tuning(b"stream_inflight", inflight) == 0
    try:
        r = np.random.default_rng(31)
        for dt, n in ((np.int64, 7_000_003), (np.float32, 9_000_011), (np.int32, 1 << 22)):
            x = GENS[dt](r, n)
            t = _cuda(x)
            o = torch.empty(n, dtype=torch.int64 if dt == np.int32 else t.dtype, device="cuda")
            device.scan(t, o, exclusive=dt == np.int32)
            _assert_array(_host(o), _expected(x, 0, dt == np.int32, np.int64 if dt == np.int32 else None), f"inflight={inflight} {dt.__name__}")
    finally:
        lib.ps_set_tuning(b"stream_inflight", prev)


@pytest.mark.parametrize("kernel", [2, 3])
def test_rounds_kernel_widening_and_chaining(ps, force_kernel, kernel):
    from paper_2312_14874_b200 import device
    force_kernel(kernel)
    flags = np.random.default_rng(2).integers(0, 2, 3_000_017, dtype=np.int32)
    out = torch.empty(flags.shape[0], dtype=torch.int64, device="cuda")
    tot = device.scan(_cuda(flags), out, exclusive=True, seed_terms=torch.tensor([7, 8], device="cuda"))
    exp = np.concatenate([[0], np.cumsum(flags[:-1], dtype=np.int64)]) + 15
    assert np.array_equal(_host(out), exp)
    assert int(tot.item()) == int(flags.sum()) + 15
    x = np.random.default_rng(3).random(2_000_000, dtype=np.float32)
    t = _cuda(x)
    device.scan(t)  # in place through the TMA ring
    ref = np.cumsum(x.astype(np.float64))
    if kernel == 2:
        assert np.array_equal(_host(t), ref.astype(np.float32))
    else:  # the stream kernel's float-pair path: within 1e-6 (bit-exact under float_exact=1)
        assert np.max(np.abs(_host(t) - ref) / ref) <= 1e-6


@pytest.mark.parametrize("kernel", [2, 3])
def test_rounds_kernel_is_deterministic(ps, force_kernel, kernel):
    from paper_2312_14874_b200 import device
    force_kernel(kernel)
    x = _cuda(np.random.default_rng(4).standard_normal(4_000_037).astype(np.float32))
    outs = []
    for _ in range(3):
        o = torch.empty_like(x)
        device.scan(x, o)
        outs.append(_host(o))
    assert all(np.array_equal(outs[0], o) for o in outs[1:])


@pytest.mark.parametrize("kernel,round_bytes", [(2, 16 << 20), (2, 48 << 20), (2, 96 << 20), (3, 0)])
def test_rounds_kernel_stress_full_size(ps, force_kernel, kernel, round_bytes):
    """Many regions x 148 CTAs, repeated: any stage-reuse or ledger race shows up
    as a persistent offset (exact integer comparison over 2^27 elements)."""
    from paper_2312_14874_b200 import device
    force_kernel(kernel, round_bytes or (48 << 20))
    flags = np.random.default_rng(7).integers(0, 2, 1 << 27, dtype=np.int32)
    ref = np.cumsum(flags, dtype=np.int64)
    x = _cuda(flags)
    out = torch.empty(flags.shape[0], dtype=torch.int64, device="cuda")
    for _ in range(3):
        tot = device.scan(x, out)
        assert int(tot.item()) == int(ref[-1])
        assert np.array_equal(_host(out), ref)


def test_seed_terms_and_total_chaining(ps):
    """Chunked scans seeded with the previous chunk's device total equal one scan
    (the pattern the multi-GPU carry and the host pipeline rely on)."""
    from paper_2312_14874_b200 import device
    r = np.random.default_rng(5)
    x = r.integers(0, 1001, 1_000_003, dtype=np.int64)
    t = _cuda(x)
    carry = torch.zeros(1, dtype=torch.int64, device="cuda")
    bounds = [0, 1, 4096, 5000, 123_457, 999_999, 1_000_003]
    for a, b in zip(bounds[:-1], bounds[1:]):
        device.scan(t[a:b], seed_terms=carry.clone(), total=carry)
    assert np.array_equal(_host(t), np.cumsum(x))
    terms = torch.tensor([5, -3, 11], dtype=torch.int64, device="cuda")
    y = _cuda(x[:10000])
    tot = device.scan(y, seed=100, seed_terms=terms)
    assert np.array_equal(_host(y), np.cumsum(x[:10000]) + 113)
    assert int(tot.item()) == int(x[:10000].sum()) + 113


def test_float32_double_accumulation_matches_reference_bitwise(ps):
    """uniform [0,1) float32 (multiples of 2^-24): every float64 partial sum is
    exact, so the GPU equals float32(cumsum(float64)) -- the reference -- bit for bit."""
    from paper_2312_14874_b200 import device
    x = np.random.default_rng(1).random(1 << 22, dtype=np.float32)
    t = _cuda(x)
    device.scan(t)
    assert np.array_equal(_host(t), np.cumsum(x.astype(np.float64)).astype(np.float32))


@pytest.mark.parametrize("rows_kernel", [1, 2])
def test_batched_rows_edge_cases(ps, rows_kernel):
    """Batched rows through both batched kernels (1 = look-back tiles, 2 = one
    CTA per row streaming 64 KiB TMA segments): single rows, tiny rows, rows
    spanning several segments, strided rows, unaligned lengths (tiles fallback)."""
    from paper_2312_14874_b200 import _lib, device
    lib = _lib.load()
    saved = lib.ps_get_tuning(b"rows_kernel")
    lib.ps_set_tuning(b"rows_kernel", rows_kernel)
    try:
        _batched_cases(device)
    finally:
        lib.ps_set_tuning(b"rows_kernel", saved)


@pytest.mark.parametrize("dynamic", [0, 1])
def test_rows_kernel_row_tickets(ps, dynamic):
    """Rows kernel with rows from the grid-wide ticket (1) or fixed shares (0): the
    same results, and the ticket counters return to zero after every launch (a
    second and third launch on the same scratch still cover every row once)."""
    from paper_2312_14874_b200 import _lib, device
    lib = _lib.load()
    saved = (lib.ps_get_tuning(b"rows_kernel"), lib.ps_get_tuning(b"rows_dynamic"))
    lib.ps_set_tuning(b"rows_kernel", 2)
    lib.ps_set_tuning(b"rows_dynamic", dynamic)
    try:
        _batched_cases(device)
        r = np.random.default_rng(12)
        for rows, cols in ((5000, 4096), (1200, 40_000)):
            x = r.integers(0, 256, (rows, cols), dtype=np.int32)
            exp = np.cumsum(x.astype(np.int64), axis=1)
            xt = _cuda(x)
            for _ in range(3):
                out = torch.full((rows, cols), -1, dtype=torch.int64, device="cuda")
                tots = torch.full((rows,), -1, dtype=torch.int64, device="cuda")
                device.scan_batched(xt, out, row_totals=tots)
                assert np.array_equal(_host(out), exp), (rows, cols, dynamic)
                assert np.array_equal(_host(tots), exp[:, -1])
    finally:
        lib.ps_set_tuning(b"rows_kernel", saved[0])
        lib.ps_set_tuning(b"rows_dynamic", saved[1])


@pytest.mark.parametrize("multi", [0, 1])
def test_rows_kernel_short_rows(ps, multi):
    """Rows of at most half a buffer: several rows per buffer (multi=1, segmented
    chunk scan per row) or one row per buffer (multi=0); seeds, totals, exclusive,
    partial last items, every value dtype."""
    from paper_2312_14874_b200 import _lib, device
    lib = _lib.load()
    saved = (lib.ps_get_tuning(b"rows_kernel"), lib.ps_get_tuning(b"rows_multi"))
    lib.ps_set_tuning(b"rows_kernel", 2)
    lib.ps_set_tuning(b"rows_multi", multi)
    try:
        r = np.random.default_rng(13)
        for rows, cols in ((5000, 3000), (3001, 12), (2000, 8192), (1999, 4100), (301, 1028), (7, 4)):
            x = r.integers(0, 256, (rows, cols), dtype=np.int32)
            seeds = torch.arange(rows, dtype=torch.int64, device="cuda") * 7
            inc = np.cumsum(x.astype(np.int64), axis=1) + (np.arange(rows) * 7)[:, None]
            for excl in (False, True):
                out = torch.full((rows, cols), -1, dtype=torch.int64, device="cuda")
                tots = torch.full((rows,), -1, dtype=torch.int64, device="cuda")
                device.scan_batched(_cuda(x), out, exclusive=excl, row_seeds=seeds, row_totals=tots)
                exp = inc if not excl else np.concatenate([(np.arange(rows) * 7)[:, None], inc[:, :-1]], axis=1)
                assert np.array_equal(_host(out), exp), (rows, cols, excl, multi)
                assert np.array_equal(_host(tots), inc[:, -1]), (rows, cols, multi)
        for dt in (np.float32, np.int64, np.uint32, np.float64):
            for rows, cols in ((3000, 1000), (500, 2052)):
                x = GENS[dt](r, rows * cols).reshape(rows, cols)
                out = torch.empty_like(_cuda(x))
                tots = torch.empty(rows, dtype=device.acc_dtype(x.dtype), device="cuda")
                device.scan_batched(_cuda(x), out, row_totals=tots)
                for i in (0, 1, rows // 2, rows - 1):
                    _assert_array(_host(out[i]), _expected(x[i]), f"{dt.__name__} row {i} {rows}x{cols}")
    finally:
        lib.ps_set_tuning(b"rows_kernel", saved[0])
        lib.ps_set_tuning(b"rows_multi", saved[1])


@pytest.mark.parametrize("row_lead", [0, 1])
def test_tiles_rows_unaligned_lengths(ps, row_lead):
    """Batched rows whose length is not a multiple of 16 bytes take the look-back
    tiles kernel; with row_lead each row's tile grid starts on its own 32-byte
    boundary (vector accesses inside, masked edges).  Strided and offset views,
    every dtype pair family, seeds, totals, exclusive."""
    from paper_2312_14874_b200 import _lib, device
    lib = _lib.load()
    saved = lib.ps_get_tuning(b"tiles_row_lead")
    lib.ps_set_tuning(b"tiles_row_lead", row_lead)
    try:
        r = np.random.default_rng(14)
        for rows, cols, ld, off in ((300, 16383, 16383, 0), (257, 16385, 16390, 3), (1000, 250, 250, 0),
                                    (64, 70_001, 70_001, 1), (999, 13, 13, 5), (40, 8191, 8200, 2),
                                    (5000, 1, 1, 0), (3000, 2047, 2047, 1), (700, 2049, 2049, 0)):
            x = r.integers(0, 256, (rows * ld + off,), dtype=np.int32)
            xv = x[off:].reshape(rows, ld)[:, :cols]
            xt = _cuda(x)[off:].reshape(rows, ld)[:, :cols]
            seeds = torch.arange(rows, dtype=torch.int64, device="cuda") * 3
            inc = np.cumsum(xv.astype(np.int64), axis=1) + (np.arange(rows) * 3)[:, None]
            for excl in (False, True):
                out = torch.full((rows, cols), -1, dtype=torch.int64, device="cuda")
                tots = torch.full((rows,), -1, dtype=torch.int64, device="cuda")
                device.scan_batched(xt, out, exclusive=excl, row_seeds=seeds, row_totals=tots)
                exp = inc if not excl else np.concatenate([(np.arange(rows) * 3)[:, None], inc[:, :-1]], axis=1)
                assert np.array_equal(_host(out), exp), (rows, cols, ld, off, excl, row_lead)
                assert np.array_equal(_host(tots), inc[:, -1]), (rows, cols, ld, off, row_lead)
            # no seeds: short contiguous rows go through the uniform-segment scan
            plain = np.cumsum(xv.astype(np.int64), axis=1)
            for excl in (False, True):
                out = torch.full((rows, cols), -1, dtype=torch.int64, device="cuda")
                tots = torch.full((rows,), -1, dtype=torch.int64, device="cuda")
                device.scan_batched(xt, out, exclusive=excl, row_totals=tots)
                exp = plain if not excl else plain - xv
                assert np.array_equal(_host(out), exp), ("noseed", rows, cols, ld, off, excl, row_lead)
                assert np.array_equal(_host(tots), plain[:, -1]), ("noseed", rows, cols, ld, off, row_lead)
        for dt in (np.float32, np.int64, np.uint32):
            for rows, cols in ((300, 5001), (50, 33_333), (2000, 777)):
                x = GENS[dt](r, rows * cols).reshape(rows, cols)
                out = torch.empty_like(_cuda(x))
                device.scan_batched(_cuda(x), out)
                for i in (0, 1, rows // 2, rows - 1):
                    _assert_array(_host(out[i]), _expected(x[i]), f"{dt.__name__} row {i} {rows}x{cols}")
    finally:
        lib.ps_set_tuning(b"tiles_row_lead", saved)


def _batched_cases(device):
    r = np.random.default_rng(8)
    for rows, cols, ld in ((1, 1, 1), (3, 5, 8), (7, 8192, 8192), (5, 8193, 8200), (64, 100_000, 100_000),
                           (2, 0, 4), (300, 16384, 16384), (301, 16388, 16400), (1000, 4, 4), (40, 200_000, 200_064)):
        x = r.integers(0, 256, (rows, ld), dtype=np.int32)
        xt = _cuda(x)[:, :cols]
        out = torch.empty((rows, cols), dtype=torch.int64, device="cuda")
        seeds = torch.arange(rows, dtype=torch.int64, device="cuda") * 1000
        tots = torch.empty(rows, dtype=torch.int64, device="cuda")
        for excl in (False, True):
            device.scan_batched(xt, out, exclusive=excl, row_seeds=seeds, row_totals=tots)
            inc = np.cumsum(x[:, :cols].astype(np.int64), axis=1) + (np.arange(rows) * 1000)[:, None]
            exp = inc if not excl else np.concatenate([(np.arange(rows) * 1000)[:, None], inc[:, :-1]], axis=1)
            if cols:
                assert np.array_equal(_host(out), exp), (rows, cols, excl)
            assert np.array_equal(_host(tots), inc[:, -1] if cols else np.arange(rows) * 1000)
    for dt in (np.float32, np.int64, np.uint32):
        for rows, cols in ((300, 16384), (40, 70_000)):
            x = GENS[dt](r, rows * cols).reshape(rows, cols)
            out = torch.empty_like(_cuda(x))
            tots = torch.empty(rows, dtype=device.acc_dtype(x.dtype), device="cuda")
            device.scan_batched(_cuda(x), out, row_totals=tots)
            for i in (0, rows // 2, rows - 1):
                _assert_array(_host(out[i]), _expected(x[i]), f"{dt.__name__} row {i} {rows}x{cols}")


def test_segmented_distributions(ps):
    """CSR segmented scan over segment-length distributions that exercise the tile ->
    segment pre-pass (galloping search from the uniform guess) and both offset paths
    (cached in shared memory, and tiles with more than SEG_CACHE segments): long
    uniform, geometric (skewed), runs of empty segments, length-1 segments, an
    unaligned view; totals and exclusive; int32 -> int64 and float32."""
    from paper_2312_14874_b200 import device
    r = np.random.default_rng(21)
    n = 3_000_003
    cases = {
        "uniform": np.sort(r.integers(0, n + 1, 300)),
        "geometric": np.cumsum(r.geometric(1 / 40, 200_000)),
        "empties": np.sort(np.concatenate([r.integers(0, n + 1, 5000), np.repeat(r.integers(0, n + 1, 50), 200)])),
        "ones": np.arange(1, n),
        "few": np.array([n // 2]),
    }
    for name, cuts in cases.items():
        cuts = cuts[(cuts > 0) & (cuts < n)]
        offs = np.concatenate([[0], cuts, [n]]).astype(np.int64)
        nseg = len(offs) - 1
        x = r.integers(0, 1000, n + 1, dtype=np.int32)
        for view in (False, True):
            xs = x[1:] if view else x[:n]
            xt = _cuda(x)[1:] if view else _cuda(x)[:n]
            for excl in (False, True):
                out = torch.empty(n, dtype=torch.int64, device="cuda")
                tots = torch.empty(nseg, dtype=torch.int64, device="cuda")
                device.scan_segmented(xt, _cuda(offs), out, exclusive=excl, seg_totals=tots)
                c = np.cumsum(xs.astype(np.int64))
                starts = np.repeat(offs[:-1], np.diff(offs))
                before = np.where(starts > 0, c[np.maximum(starts - 1, 0)], 0)
                inc = c - before
                exp = inc - xs if excl else inc
                assert np.array_equal(_host(out), exp), (name, view, excl)
                ends = offs[1:] - 1
                exp_tot = np.where(np.diff(offs) > 0, c[np.maximum(ends, 0)] - np.where(offs[:-1] > 0, c[np.maximum(offs[:-1] - 1, 0)], 0), 0)
                assert np.array_equal(_host(tots), exp_tot), (name, view)
        f = r.random(n, dtype=np.float32)
        out = torch.empty(n, dtype=torch.float32, device="cuda")
        device.scan_segmented(_cuda(f), _cuda(offs), out)
        c = np.cumsum(f.astype(np.float64))
        starts = np.repeat(offs[:-1], np.diff(offs))
        before = np.where(starts > 0, c[np.maximum(starts - 1, 0)], 0.0)
        np.testing.assert_allclose(_host(out), (c - before).astype(np.float32), rtol=1e-5, atol=1e-4, err_msg=name)


def test_shared_scratch_segmented_then_stream(ps, force_kernel):
    """One scratch shared by a segmented scan and a later stream-kernel scan (the
    C ABI allows it): the segmented pre-pass's tile -> segment words sit where the
    stream kernel's region descriptors go, and must never pass for a published
    descriptor of a later epoch (segment 9 == (epoch 2 << 2) | 1 would, stored
    plainly).  Integer ledgers poll early, so a stale match would be taken."""
    from paper_2312_14874_b200 import _lib
    lib = _lib.load()
    force_kernel(3)
    n = 1 << 24
    r = np.random.default_rng(23)
    x = _cuda(r.integers(0, 100, n, dtype=np.int32))
    # a 100000-element segmented scan (13 tiles) puts its tile -> segment words at scratch
    # offset 512, i.e. on region 0's descriptors of the stream kernel; segment 9 holds
    # tiles 1..12, and 9 == (2 << 2) | 1 is a "published" tag for epoch 2
    m = 100_000
    offs = _cuda(np.concatenate([np.arange(10), [m]]).astype(np.int64))
    sbytes = max(lib.ps_scan_segmented_scratch_bytes(m, 1, 2), lib.ps_scan_scratch_bytes(n, 1, 2))
    for trial in range(3):
        scratch = torch.zeros(sbytes, dtype=torch.uint8, device="cuda")
        seg_out = torch.empty(m, dtype=torch.int64, device="cuda")
        assert lib.ps_scan_segmented(x.data_ptr(), seg_out.data_ptr(), m, offs.data_ptr(), 10, 1, 2, 0, None,
                                     scratch.data_ptr(), sbytes, 1, None) == 0
        out = torch.empty(n, dtype=torch.int64, device="cuda")
        tot = torch.empty(1, dtype=torch.int64, device="cuda")
        assert lib.ps_scan(x.data_ptr(), out.data_ptr(), n, 1, 2, 0, 0, None, 0, tot.data_ptr(),
                           scratch.data_ptr(), sbytes, 2, None) == 0
        torch.cuda.synchronize()
        exp = np.cumsum(_host(x).astype(np.int64))
        assert np.array_equal(_host(out), exp), trial
        assert int(tot.item()) == int(exp[-1])


def test_segmented(ps):
    from paper_2312_14874_b200 import device
    r = np.random.default_rng(9)
    for n, nseg in ((0, 1), (1, 1), (10, 3), (50_000, 1), (100_000, 7), (300_001, 1000), (40_000, 40_000)):
        x = r.integers(0, 100, n, dtype=np.int32)
        cuts = np.sort(r.integers(0, n + 1, nseg - 1)) if nseg > 1 else np.array([], np.int64)
        offs = np.concatenate([[0], cuts, [n]]).astype(np.int64)
        for excl in (False, True):
            xt = _cuda(x)
            out = torch.empty(n, dtype=torch.int64, device="cuda")
            tots = torch.empty(nseg, dtype=torch.int64, device="cuda")
            device.scan_segmented(xt, _cuda(offs), out, exclusive=excl, seg_totals=tots)
            exp = np.empty(n, np.int64)
            exp_tot = np.zeros(nseg, np.int64)
            for s in range(nseg):
                seg = x[offs[s]:offs[s + 1]].astype(np.int64)
                c = np.cumsum(seg)
                exp[offs[s]:offs[s + 1]] = c - seg if excl else c
                exp_tot[s] = seg.sum()
            assert np.array_equal(_host(out), exp), (n, nseg, excl)
            assert np.array_equal(_host(tots), exp_tot), (n, nseg)


def test_shift_right_in_place_large(ps):
    from paper_2312_14874_b200 import device
    x = np.random.default_rng(2).integers(0, 2**40, 1_000_001, dtype=np.int64)
    t = _cuda(x)
    last = device.shift_right(t, identity=-5)
    assert int(last.item()) == int(x[-1])
    assert np.array_equal(_host(t), np.concatenate([[-5], x[:-1]]))


def test_reduce_and_add_offset_large(ps):
    from paper_2312_14874_b200 import device
    r = np.random.default_rng(4)
    for dt in (np.int64, np.float32, np.uint32, np.int32):
        x = GENS[dt](r, 3_000_017)
        for s in (0, 1, 3):
            t = _cuda(x)[s:]
            tot = device.reduce(t, seed=2)
            if x.dtype.kind == "f":
                assert abs(tot.item() - (x[s:].astype(np.float64).sum() + 2)) < 1e-6 * x.size
            elif dt == np.uint32:
                assert int(tot.cpu().view(torch.int64).item()) == int(x[s:].astype(np.uint64).sum()) + 2
            else:
                assert int(tot.item()) == int(x[s:].astype(np.int64).sum()) + 2
            device.add_offset(t, 3)
            exp = (x[s:].astype(np.float64) + 3).astype(dt) if x.dtype.kind == "f" else (x[s:] + dt(3)).astype(dt)
            assert np.array_equal(_host(t), exp), dt


def test_reduce_is_deterministic(ps):
    from paper_2312_14874_b200 import device
    x = _cuda(np.random.default_rng(6).standard_normal(10_000_019).astype(np.float32))
    vals = {device.reduce(x).item() for _ in range(5)}
    assert len(vals) == 1


def test_host_pipeline_end_to_end(ps):
    """ps_scan_host: pinned and pageable host buffers, chunk boundaries, seeds."""
    from paper_2312_14874_b200 import device
    r = np.random.default_rng(12)
    x = r.integers(0, 101, 3_000_001, dtype=np.int64)
    for chunk in (1 << 16, 1_000_000, 1 << 22):
        pinned_in = torch.from_numpy(x).pin_memory()
        pinned_out = torch.empty_like(pinned_in).pin_memory()
        tot = device.scan_host(pinned_in, pinned_out, seed=5, chunk_elems=chunk)
        assert np.array_equal(pinned_out.numpy(), np.cumsum(x) + 5)
        assert tot == int(x.sum()) + 5
        y = x.copy()
        tot = device.scan_host(y, exclusive=True, chunk_elems=chunk)  # pageable, in place
        assert np.array_equal(y, np.concatenate([[0], np.cumsum(x)[:-1]]))
        assert tot == int(x.sum())
    f = r.random(2_000_003, dtype=np.float32)
    g = np.empty(f.shape[0], np.float64)
    device.scan_host(f, g, chunk_elems=1 << 18)
    assert np.array_equal(g, np.cumsum(f.astype(np.float64)))


def test_errors_match_reference(ps):
    t = torch.zeros(4, dtype=torch.int64, device="cuda")
    with pytest.raises(ValueError):
        ps.sequential_inclusive_scan(t, ps.Span(2, 3))
    with pytest.raises(ValueError):
        ps.horizontal_scan(t, ps.full_span(t), 0, w=5)
    with pytest.raises(ValueError):
        ps.tree_scan(torch.zeros(48, dtype=torch.uint32, device="cuda"), ps.Span(0, 48), 0, 16)
    with pytest.raises(ValueError):
        ps.ScanRequest(data=t, out=t)
    with pytest.raises(ValueError):
        ps.sequential_inclusive_scan(torch.zeros(4, dtype=torch.int16, device="cuda"), ps.Span(0, 4))


def test_vertical_pass_functions(ps):
    """The reference's step-level KATs (test_simd.py:109-183) against the GPU batched kernels."""
    from paper_2312_14874_b200.simd import (exclusive_offsets, vertical_scan_pass1_accumulate,
                                            vertical_scan_pass1_scan, vertical_scan_pass2_increment,
                                            vertical_scan_pass2_scan)
    for where in ("numpy", "cuda"):
        data = np.array([1, 2, 3, 4, 5, 6, 7, 8], dtype=np.uint32)
        d = _cuda(data) if where == "cuda" else data.copy()
        totals = np.zeros(2, dtype=np.uint64)
        vertical_scan_pass1_scan(d, ps.full_span(d), 0, totals)
        assert (_host(d) if where == "cuda" else d).tolist() == [1, 3, 6, 10, 5, 11, 18, 26]
        assert totals.tolist() == [10, 26]
        vertical_scan_pass2_increment(d, ps.full_span(d), exclusive_offsets(totals, np.uint64(0)))
        assert (_host(d) if where == "cuda" else d).tolist() == [1, 3, 6, 10, 15, 21, 28, 36]

        d = _cuda(data) if where == "cuda" else data.copy()
        vertical_scan_pass1_accumulate(d, ps.full_span(d), totals)
        assert totals.tolist() == [10, 26]
        vertical_scan_pass2_scan(d, ps.full_span(d), exclusive_offsets(totals, np.uint64(0)))
        assert (_host(d) if where == "cuda" else d).tolist() == [1, 3, 6, 10, 15, 21, 28, 36]

        d = np.array([3, 4, 5, 6], dtype=np.uint32)
        totals = np.zeros(4, dtype=np.uint64)
        dd = _cuda(d) if where == "cuda" else d
        vertical_scan_pass1_scan(dd, ps.full_span(dd), 100, totals)
        assert (_host(dd) if where == "cuda" else dd).tolist() == [103, 4, 5, 6]
        assert totals.tolist() == [103, 4, 5, 6]


# ---- BASELINE.json configs at full size ---------------------------------------------------------

def test_cfg1_full(ps, oracle_lib):
    x = np.random.default_rng(0).integers(0, 101, 2**24, dtype=np.int64)
    want = x.copy()
    wt = oracle_lib.scan(want, 0, want.shape[0], 0)  # the reference algorithm, restated
    t = _cuda(x)
    total = ps.sequential_inclusive_scan(t, ps.full_span(t))
    assert np.array_equal(_host(t), want)
    assert total == wt


@pytest.mark.parametrize("float_exact", [0, 1])
def test_cfg2_full(ps, float_exact):
    """cfg2 at full size.  float_exact=1: float64 per element, bit-exact (the
    BASELINE draw's float64 partial sums are exact).  Default (0): float32
    in-chunk scans with a float-pair carry -- within 1e-6 of the reference
    (BASELINE allows 1e-4); the total is float64 either way."""
    from paper_2312_14874_b200 import _lib
    lib = _lib.load()
    x = np.random.default_rng(1).random(2**28, dtype=np.float32)
    ref = np.cumsum(x.astype(np.float64))
    t = _cuda(x)
    prev = lib.ps_get_tuning(b"float_exact")
    assert lib.ps_set_tuning(b"float_exact", float_exact) == 0
    try:
        total = ps.sequential_inclusive_scan(t, ps.full_span(t))
    finally:
        lib.ps_set_tuning(b"float_exact", prev)
    got = _host(t)
    rel = np.abs(got.astype(np.float64) - ref) / np.maximum(ref, 1e-30)
    if float_exact:
        assert np.array_equal(got, ref.astype(np.float32))  # exact partial sums -> bit-exact
    assert rel.max() <= 1e-6 and total == ref[-1], rel.max()


@pytest.mark.parametrize("gen", ["uniform", "normal", "mixed_magnitude", "seeded_negative"])
def test_float32_pair_path_accuracy(ps, force_kernel, gen):
    """The stream kernel's float32 fast path engages only on nonnegative chunks
    under a carry >= 64x the chunk sum; signed data, huge dynamic range and a
    negative seed must still meet the reference within 1e-6 relative (or 1e-6
    of the running magnitude where the sum crosses zero)."""
    from paper_2312_14874_b200 import device
    force_kernel(3)
    r = np.random.default_rng(77)
    n = 9_000_011
    if gen == "uniform":
        x, seed = r.random(n, dtype=np.float32), 0.0
    elif gen == "normal":
        x, seed = r.standard_normal(n).astype(np.float32), 0.0
    elif gen == "mixed_magnitude":
        x, seed = (r.random(n) * 10.0 ** r.integers(-6, 7, n)).astype(np.float32), 0.0
    else:
        x, seed = r.random(n, dtype=np.float32), -1e6
    t = _cuda(x)
    o = torch.empty_like(t)
    device.scan(t, o, seed=seed)
    got = _host(o).astype(np.float64)
    ref = np.cumsum(x.astype(np.float64)) + seed
    scale = np.maximum(np.abs(ref), np.maximum.accumulate(np.abs(ref)) * 1e-3) if gen != "uniform" else np.abs(ref)
    err = np.abs(got - ref) / np.maximum(scale, 1e-30)
    assert err.max() <= 1e-6, (gen, err.max())


def test_cfg3_full(ps):
    from paper_2312_14874_b200 import device
    flags = np.random.default_rng(2).integers(0, 2, 2**28, dtype=np.int32)
    t = _cuda(flags)
    out = torch.empty(2**28, dtype=torch.int64, device="cuda")
    total = device.scan(t, out, exclusive=True)
    got = _host(out)
    assert int(total.item()) == int(flags.sum())
    assert got[0] == 0
    assert np.array_equal(got[1:], np.cumsum(flags[:-1], dtype=np.int64))


def test_cfg4_full(ps):
    from paper_2312_14874_b200 import device
    x = np.random.default_rng(3).integers(0, 256, (16384, 16384), dtype=np.int32)
    t = _cuda(x)
    out = torch.empty((16384, 16384), dtype=torch.int64, device="cuda")
    device.scan_batched(t, out)
    got = _host(out)
    assert np.array_equal(got, np.cumsum(x, axis=1, dtype=np.int64))


def test_cfg5_full_properties(ps):
    """2^31 int64 (16 GB in + 16 GB out) on one GPU: generated on the device;
    checked through size-independent properties -- first differences give the
    input back, the total equals an independent reduction, and sampled windows
    match numpy continued from the carry."""
    from paper_2312_14874_b200 import device
    n = 2**31
    if torch.cuda.get_device_properties(0).total_memory < 40 * 2**30:
        pytest.skip("needs > 40 GB of device memory")
    g = torch.Generator(device="cuda").manual_seed(4)
    x = torch.randint(0, 1001, (n,), dtype=torch.int64, device="cuda", generator=g)
    out = torch.empty_like(x)
    total = device.scan(x, out)
    red = device.reduce(x)
    assert int(total.item()) == int(red.item())
    assert int(out[-1].item()) == int(total.item())
    step = 1 << 28
    for a in range(0, n, step):
        b = min(n, a + step)
        d = out[a + 1:b] - out[a:b - 1]
        assert torch.equal(d, x[a + 1:b])
    assert int(out[0].item()) == int(x[0].item())
    xs = x[:1 << 20].cpu().numpy()
    assert np.array_equal(out[:1 << 20].cpu().numpy(), np.cumsum(xs))
    for a in (n // 3, n - (1 << 20)):
        w = x[a:a + (1 << 20)].cpu().numpy()
        carry = int(out[a - 1].item())
        assert np.array_equal(out[a:a + (1 << 20)].cpu().numpy(), np.cumsum(w) + carry)


def test_cfg5_baseline_draw_bit_exact(ps):
    """cfg5 on the exact BASELINE.json draw (np.random.default_rng(4), 2^31 int64 in
    [0, 1000]): the whole output chunk-wise against np.cumsum continued with the carry
    (== the reference's `_scan_kernel`, core.py:86-92, below 2^53) and the returned total
    against the value the survey recorded from the reference itself."""
    import psutil
    import bench
    from paper_2312_14874_b200 import device
    if torch.cuda.get_device_properties(0).total_memory < 40 * 2**30:
        pytest.skip("needs > 40 GB of device memory")
    if psutil.virtual_memory().available < 24 * 2**30:
        pytest.skip("needs 16 GiB of host memory for the BASELINE draw")
    cfg = bench.CONFIGS["cfg5"]
    xh = bench.host_input(cfg)
    assert xh.shape == (2**31,) and xh.dtype == np.int64
    x = torch.empty(2**31, dtype=torch.int64, device="cuda")
    step = 1 << 28
    for a in range(0, 2**31, step):
        x[a:a + step].copy_(torch.from_numpy(xh[a:a + step]))
    out = torch.empty_like(x)
    total = device.scan(x, out)
    assert int(total.item()) == bench.KNOWN_TOTALS["cfg5"] == 1073746006907
    res = bench.verify_host(cfg, xh, out)  # raises on the first differing element
    assert res["bit_exact"] and res["total"] == 1073746006907


@pytest.mark.parametrize("din,dout", [(np.int32, np.int64), (np.int64, np.int64), (np.float32, np.float32)])
def test_stream_kernel_input_and_output_at_different_phases(ps, din, dout):
    """Inputs >= 32 MiB whose input and output sit at different 32-byte phases run on the stream
    kernel with the tile grid aligned to the OUTPUT: bulk copies where the input's 16-byte phase
    fits, the reducer warps' element-wise cp.async otherwise.  A spread of element-offset pairs."""
    from paper_2312_14874_b200 import device
    r = np.random.default_rng(41)
    n = (9 << 20) + 4321 if np.dtype(din).itemsize == 4 else (5 << 20) + 99
    fl = np.dtype(din).kind == "f"
    acc = np.float64 if fl else np.int64
    xh = (r.integers(0, 1024, n + 8) / 1024.0).astype(din) if fl else r.integers(-100, 300, n + 8).astype(din)
    xd = torch.from_numpy(xh).cuda()
    od = torch.empty(n + 8, dtype=getattr(torch, np.dtype(dout).name), device="cuda")
    for oi, oo in ((0, 1), (1, 0), (3, 2), (5, 0), (2, 7), (7, 7), (4, 1)):
        excl = bool((oi + oo) & 1)
        o = od[oo:oo + n]
        o.zero_()
        tot = device.scan(xd[oi:oi + n], o, exclusive=excl, seed=3)
        c = np.cumsum(xh[oi:oi + n].astype(acc)) + acc(3)
        want = (np.concatenate([[acc(3)], c[:-1]]) if excl else c).astype(dout)  # exact on the 2^-10 grid
        assert np.array_equal(o.cpu().numpy(), want), (din, oi, oo, excl)
        assert tot.cpu().numpy().view(acc)[0] == c[-1]


def test_cuda_graph_replays(ps):
    """Scans captured in a CUDA graph and replayed several times over changing input
    contents: every replay starts from a zeroed scratch (the epochs are baked into the
    graph), so no replay can take a previous replay's descriptors for its own."""
    from paper_2312_14874_b200 import device
    r = np.random.default_rng(29)
    n_big, n_small = 9_000_011, 300_007
    big = torch.empty(n_big, dtype=torch.int64, device="cuda")
    small = torch.empty(n_small, dtype=torch.float32, device="cuda")
    rows = torch.empty((3000, 5001), dtype=torch.int32, device="cuda")
    flags = torch.empty(n_small, dtype=torch.int32, device="cuda")
    ob, os_, orow = torch.empty_like(big), torch.empty_like(small), torch.empty((3000, 5001), dtype=torch.int64, device="cuda")
    osel = torch.empty(n_small, dtype=torch.float32, device="cuda")
    cnt = torch.empty(1, dtype=torch.int64, device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())

    def work():
        device.scan(big, ob)
        device.scan(small, os_)
        device.scan_batched(rows, orow, exclusive=True)
        device.select(small, flags, osel, count=cnt)

    with torch.cuda.stream(s):
        work()  # warm-up: scratch sized on the capture stream
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        work()
    for rep in range(4):
        xb = r.integers(0, 1000, n_big, dtype=np.int64)
        xs = r.random(n_small, dtype=np.float32)
        xr = r.integers(0, 256, (3000, 5001), dtype=np.int32)
        xf = r.integers(0, 2, n_small, dtype=np.int32)
        big.copy_(torch.from_numpy(xb))
        small.copy_(torch.from_numpy(xs))
        rows.copy_(torch.from_numpy(xr))
        flags.copy_(torch.from_numpy(xf))
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(_host(ob), np.cumsum(xb)), rep
        np.testing.assert_allclose(_host(os_), np.cumsum(xs.astype(np.float64)).astype(np.float32), rtol=1e-6)
        inc = np.cumsum(xr.astype(np.int64), axis=1)
        assert np.array_equal(_host(orow), inc - xr), rep
        k = int(cnt.item())
        assert k == int(xf.sum()) and np.array_equal(_host(osel)[:k], xs[xf != 0]), rep


@pytest.mark.parametrize("blocks", [0, 1])
def test_reduce_block_tickets(ps, blocks):
    """ps_reduce with blocks from a ticket (1) or grid-stride shares (0): exact for
    integers, run-to-run identical for floats (blocks fold in block order whichever
    CTA reduced them), unaligned heads and tails, seeds, repeated launches."""
    from paper_2312_14874_b200 import _lib, device
    lib = _lib.load()
    saved = lib.ps_get_tuning(b"reduce_blocks")
    lib.ps_set_tuning(b"reduce_blocks", blocks)
    try:
        r = np.random.default_rng(41)
        for n, off in ((1, 0), (7, 3), (100_003, 1), (5_000_011, 5), (1 << 24, 0), ((1 << 26) + 3, 2)):
            x = r.integers(-1000, 1000, n + off, dtype=np.int64)
            t = _cuda(x)[off:]
            for rep in range(2):
                assert int(device.reduce(t, seed=7).item()) == int(x[off:].sum()) + 7, (n, off)
            f = r.random(n + off, dtype=np.float32)
            ft = _cuda(f)[off:]
            a, b = float(device.reduce(ft).item()), float(device.reduce(ft).item())
            assert a == b
            np.testing.assert_allclose(a, f[off:].astype(np.float64).sum(), rtol=1e-9)
    finally:
        lib.ps_set_tuning(b"reduce_blocks", saved)
