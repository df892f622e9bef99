"""scripts/shape_sweep.py -- dev tool: HBM fraction of the scan paths over shapes that
the BASELINE configs do not cover (small 1-D, unaligned rows, segmented)."""
import sys

import torch

sys.path.insert(0, ".")
import os  # noqa: E402

from paper_2312_14874_b200 import _build  # noqa: E402

if os.environ.get("LIB"):  # A/B against another build of the library
    _build.LIB_PATH = os.environ["LIB"]
    _build.up_to_date = lambda: True
from paper_2312_14874_b200 import device  # noqa: E402

PEAK = 6551.0


def t(fn, K=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(K):
            fn()
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b) / K * 1e3)
    return best


def report(name, us, byt):
    print(f"{name:42s} {us:9.1f} us  {byt / us / 1e3:7.0f} GB/s  ({byt / us / 1e3 / PEAK:.3f})", flush=True)


for n, dt, dto in ((1 << 18, torch.int64, torch.int64), (1 << 20, torch.int64, torch.int64),
                   (1 << 21, torch.int64, torch.int64), (1 << 22, torch.float32, torch.float32),
                   (1 << 23, torch.float32, torch.float32), (1 << 22, torch.int32, torch.int64),
                   (3 << 20, torch.int64, torch.int64), ((1 << 24) + 7, torch.int64, torch.int64),
                   ((1 << 28) + 3, torch.float32, torch.float32)):
    x = torch.randint(0, 100, (n,), device="cuda").to(dt)
    o = torch.empty(n, dtype=dto, device="cuda")
    report(f"1-D n={n} {dt}->{dto}", t(lambda: device.scan(x, o)), n * (x.element_size() + o.element_size()))
# unaligned start (view at +1 element)
x = torch.randint(0, 100, ((1 << 26) + 1,), device="cuda")
o = torch.empty_like(x)
report("1-D 2^26 int64, in/out offset +1", t(lambda: device.scan(x[1:], o[1:])), (1 << 26) * 16)
report("1-D 2^26 int64, out offset +1 only", t(lambda: device.scan(x[:-1], o[1:])), (1 << 26) * 16)
for rows, cols in ((16384, 16383), (16384, 16385), (4096, 65537), (65536, 3001), (1 << 20, 250)):
    x = torch.randint(0, 256, (rows, cols), device="cuda", dtype=torch.int32)
    o = torch.empty((rows, cols), dtype=torch.int64, device="cuda")
    report(f"rows {rows}x{cols} i32->i64", t(lambda: device.scan_batched(x, o)), rows * cols * 12)
for n, nseg in ((1 << 28, 1 << 14), (1 << 28, 1 << 20), (1 << 26, 1 << 24)):
    x = torch.randint(0, 256, (n,), device="cuda", dtype=torch.int32)
    offs = torch.sort(torch.randint(0, n + 1, (nseg + 1,), device="cuda"))[0]
    offs[0], offs[-1] = 0, n
    o = torch.empty(n, dtype=torch.int64, device="cuda")
    report(f"segmented n={n} nseg={nseg} i32->i64", t(lambda: device.scan_segmented(x, offs, o)),
           n * 12 + (nseg + 1) * 8)
