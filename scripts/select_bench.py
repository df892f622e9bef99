"""Time ps_select (stream compaction / stable partition) at 2^28 elements (dev tool).
Prints per-launch kernel times with CUDA events and the effective bandwidth against the
single-pass algorithmic bytes (flags + values read once, output written once)."""
import sys

import torch

sys.path.insert(0, ".")
import os  # noqa: E402

from paper_2312_14874_b200 import _build  # noqa: E402

if os.environ.get("LIB"):  # A/B against another build of the library
    _build.LIB_PATH = os.environ["LIB"]
    _build.up_to_date = lambda: True
from paper_2312_14874_b200 import _lib  # noqa: E402
from paper_2312_14874_b200 import device as dev  # noqa: E402

if os.environ.get("INFL"):  # the single-pass kernel's bound on outstanding region loads
    _lib.load().ps_set_tuning(b"stream_inflight", int(os.environ["INFL"]))

n = 1 << 28
g = torch.Generator(device="cuda").manual_seed(5)
for fdt, vdt, p in [(torch.int32, torch.int32, 0.5), (torch.uint8, torch.int32, 0.5), (torch.uint8, torch.int64, 0.5),
                    (torch.int32, torch.int32, 0.05), (torch.int32, torch.int32, 0.95)]:
    f = (torch.rand(n, device="cuda", generator=g) < p).to(fdt)
    v = torch.arange(n, dtype=vdt, device="cuda")
    out = torch.empty_like(v)
    cnt = torch.empty(1, dtype=torch.int64, device="cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for partition in (False, True):
        for _ in range(3):
            dev.select(v, f, out, partition=partition, count=cnt)
        ts = []
        for _ in range(10):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            dev.select(v, f, out, partition=partition, count=cnt)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        t = sorted(ts)[len(ts) // 2]
        k = int(cnt.item())
        fb, vb = f.element_size(), v.element_size()
        alg = n * (fb + vb) + (n if partition else k) * vb
        single = (not partition) and fb >= 4  # ps_select's auto choice (single pass) -> flags read once
        moved = alg + (0 if single else n * fb)
        print(f"flags {str(fdt):12s} values {str(vdt):12s} p={p:<5} {'partition' if partition else 'select   '} "
              f"{'1-pass' if single else '3-launch'} "
              f"{t * 1e3:8.1f} us  alg {alg / t / 1e6:7.1f} GB/s  moved {moved / t / 1e6:7.1f} GB/s")
