"""Randomised soak test of every scan path against numpy (dev tool):

    python scripts/soak.py [seconds]

Random dtype pairs, sizes (1 .. 2^27), unaligned views, inclusive/exclusive,
seeds, forced kernels (look-back / L2 rounds / stream / auto), batched rows
(both kernels, row tickets, short rows, per-row tile grids, seeds and totals),
CSR segmented scans, compaction, reduce and add-offset, with and without stall
injection.  Prints a line
per 100 cases and exits non-zero on the first mismatch (with its parameters)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2312_14874_b200 import _lib, device as dev  # noqa: E402

lib = _lib.load()
PAIRS = [(np.int32, np.int32), (np.int32, np.int64), (np.int64, np.int64), (np.uint32, np.uint64),
         (np.uint32, np.uint32), (np.float32, np.float32), (np.float32, np.float64), (np.float64, np.float64)]
rng = np.random.default_rng(int(time.time()))
deadline = time.time() + (float(sys.argv[1]) if len(sys.argv) > 1 else 300)
cases = 0


def ref_scan(a, dout, exclusive, seed):
    acc = np.float64 if np.dtype(dout).kind == "f" else (np.uint64 if np.dtype(a.dtype).kind == "u" else np.int64)
    c = np.cumsum(a.astype(acc)) + acc(seed) if a.size else np.zeros(0, acc)
    if exclusive and a.size:
        c = np.concatenate([[acc(seed)], c[:-1]])
    return c.astype(dout)


def compare(got, want, what):
    if np.dtype(want.dtype).kind == "f":
        w = want.astype(np.float64)
        rel = np.abs(got.astype(np.float64) - w) / np.maximum(np.abs(w), 1e-30)
        ok = got.size == 0 or rel.max() <= 2e-6
    else:
        ok = np.array_equal(got, want)
    if not ok:
        raise SystemExit(f"MISMATCH {what}")


while time.time() < deadline:
    din, dout = PAIRS[rng.integers(len(PAIRS))]
    n = int(rng.choice([1, 7, 4096, 8191, 100_003, 1 << 20, 3_000_001, 1 << 24, (1 << 25) + 17, 1 << 27]))
    off = int(rng.integers(0, 8))
    excl = bool(rng.integers(2))
    seed = int(rng.integers(0, 50))
    kern = int(rng.integers(0, 4))
    stall = rng.random() < 0.15
    if np.dtype(din).kind == "f":
        a = rng.random(n + off).astype(din)
    else:
        a = rng.integers(0, 100, n + off).astype(din)
    x = torch.from_numpy(a).cuda()[off:]
    out = torch.empty(n, dtype=torch.from_numpy(np.zeros(1, dout)).dtype, device="cuda")
    lib.ps_set_tuning(b"scan_kernel", kern)
    try:
        if stall:
            with dev.stall_injection(seed=cases + 1, prob=0.1, max_ns=10000):
                dev.scan(x, out, exclusive=excl, seed=seed)
        else:
            dev.scan(x, out, exclusive=excl, seed=seed)
    finally:
        lib.ps_set_tuning(b"scan_kernel", 0)
    compare(out.cpu().numpy(), ref_scan(a[off:], dout, excl, seed),
            f"scan {din.__name__}->{dout.__name__} n={n} off={off} excl={excl} seed={seed} kernel={kern} stall={stall}")
    cases += 1
    if cases % 7 == 0:  # batched rows: both kernels, row tickets, short rows, per-row tile grids
        rows = int(rng.choice([int(rng.integers(1, 700)), int(rng.integers(700, 20000))]))
        cols = int(rng.choice([int(rng.integers(1, 40000)), int(rng.integers(1, 3000))]))
        if cases % 21 == 0:  # a large batch of short rows: the flat segmented scan on the region kernel
            cols = int(rng.integers(1, 700))
            rows = (40 << 20) // (4 * cols) + int(rng.integers(0, 1000))
        b = rng.integers(0, 255, (rows, cols)).astype(np.int32)
        knobs = {b"rows_kernel": int(rng.integers(0, 3)), b"rows_dynamic": int(rng.integers(0, 2)),
                 b"rows_multi": int(rng.integers(0, 2)), b"tiles_row_lead": int(rng.integers(0, 2))}
        saved = {k: lib.ps_get_tuning(k) for k in knobs}
        for k, v in knobs.items():
            lib.ps_set_tuning(k, v)
        seeded = bool(rng.integers(2))
        seeds = torch.arange(rows, dtype=torch.int64, device="cuda") * 5 if seeded else None
        o = torch.empty((rows, cols), dtype=torch.int64, device="cuda")
        tots = torch.empty(rows, dtype=torch.int64, device="cuda")
        dev.scan_batched(torch.from_numpy(b).cuda(), o, exclusive=excl, row_seeds=seeds, row_totals=tots)
        for k, v in saved.items():
            lib.ps_set_tuning(k, v)
        want = np.cumsum(b, axis=1, dtype=np.int64) + ((np.arange(rows) * 5)[:, None] if seeded else 0)
        compare(tots.cpu().numpy(), want[:, -1], f"row totals {rows}x{cols} {knobs} seeded={seeded}")
        if excl:
            want = want - b
        compare(o.cpu().numpy(), want, f"rows {rows}x{cols} excl={excl} {knobs} seeded={seeded}")
    if cases % 5 == 0:  # CSR segmented: both kernels, dtype pairs, totals, in place, unaligned views
        m = int(rng.choice([1000, 1 << 20, 3_000_001, 9_000_013]))
        nseg = int(rng.choice([1, 10, 1000, m // 300 + 1, m // 4 + 1]))
        cuts = np.sort(rng.integers(0, m + 1, nseg - 1))  # repeated offsets = empty segments
        offs = np.concatenate([[0], cuts, [m]]).astype(np.int64)
        sdin, sdout = PAIRS[int(rng.integers(0, len(PAIRS)))]
        fl = np.dtype(sdout).kind == "f"
        acc = np.float64 if fl else (np.uint64 if np.dtype(sdin).kind == "u" else np.int64)
        # floats on a 2^-10 grid: every float64 partial sum is exact, so the cumsum-difference
        # reference below has no cancellation error and the comparison is meaningful
        v = (rng.integers(0, 1024, m) / 1024.0).astype(sdin) if np.dtype(sdin).kind == "f" else rng.integers(0, 100, m).astype(sdin)
        sk = int(rng.integers(0, 3))
        lib.ps_set_tuning(b"seg_kernel", sk)
        lead = int(rng.integers(0, 4))
        xin = torch.empty(m + lead, dtype=getattr(torch, np.dtype(sdin).name), device="cuda")[lead:]
        xin.copy_(torch.from_numpy(v))
        inplace = sdin == sdout and rng.random() < 0.3
        o = xin if inplace else torch.empty(m + lead, dtype=getattr(torch, np.dtype(sdout).name), device="cuda")[lead:]
        tots = torch.empty(nseg, dtype=getattr(torch, np.dtype(acc).name), device="cuda") if rng.random() < 0.7 else None
        dev.scan_segmented(xin, torch.from_numpy(offs).cuda(), o, exclusive=excl, seg_totals=tots)
        lib.ps_set_tuning(b"seg_kernel", 0)
        c = np.concatenate([[acc(0)], np.cumsum(v.astype(acc))]).astype(acc)
        seg_of = np.searchsorted(offs, np.arange(m), side="right") - 1
        want = ((c[:-1] if excl else c[1:]) - c[offs[seg_of]]).astype(sdout)
        what = f"segmented {np.dtype(sdin).name}->{np.dtype(sdout).name} m={m} nseg={nseg} excl={excl} kernel={sk} lead={lead} inplace={inplace}"
        compare(o.cpu().numpy(), want, what)
        if tots is not None:
            wt = (c[offs[1:]] - c[offs[:-1]]).astype(acc)
            gt = tots.cpu().numpy()
            if fl:
                ok = np.allclose(gt, wt, rtol=1e-9, atol=1e-6)
            else:
                ok = np.array_equal(gt, wt)
            if not ok:
                print("MISMATCH totals", what, flush=True)
                sys.exit(1)
    if cases % 11 == 0:  # compaction
        m = int(rng.choice([1000, 1 << 20, 5_000_000]))
        v = rng.integers(-1000, 1000, m).astype(np.int32)
        f = (rng.random(m) < rng.random()).astype(np.int32)
        lib.ps_set_tuning(b"select_kernel", int(rng.integers(0, 3)))
        o, cnt = dev.select(torch.from_numpy(v).cuda(), torch.from_numpy(f).cuda())
        lib.ps_set_tuning(b"select_kernel", 0)
        k = int(cnt.item())
        compare(o[:k].cpu().numpy(), v[f != 0], f"select m={m}")
    if cases % 5 == 0:  # reduce (block tickets) and add_offset (one CTA per 64 KiB)
        m = int(rng.choice([1, 1000, 1 << 20, 9_000_011, 1 << 26]))
        o2 = int(rng.integers(0, 8))
        v = rng.integers(-1000, 1000, m + o2).astype(np.int64)
        t = torch.from_numpy(v).cuda()[o2:]
        lib.ps_set_tuning(b"reduce_blocks", int(rng.integers(0, 2)))
        compare(np.array([int(dev.reduce(t).item())]), np.array([int(v[o2:].sum())]), f"reduce m={m} off={o2}")
        lib.ps_set_tuning(b"reduce_blocks", 1)
        lib.ps_set_tuning(b"add_chunked", int(rng.integers(0, 2)))
        dev.add_offset(t, 17)
        lib.ps_set_tuning(b"add_chunked", 1)
        compare(t.cpu().numpy(), v[o2:] + 17, f"add_offset m={m} off={o2}")
    if cases % 100 == 0:
        print(f"{cases} cases ok", flush=True)
print(f"soak ok: {cases} cases")
