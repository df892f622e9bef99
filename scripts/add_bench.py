"""scripts/add_bench.py -- dev tool: ps_add_offset (sequential_increment, scan-then-fixup
phase 2) in place, one CTA per 64 KiB (add_chunked=1) vs grid-stride shares (0)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2312_14874_b200 import _lib, device as dev  # noqa: E402

lib = _lib.load()
for dt, n in ((torch.float32, 1 << 28), (torch.int64, 1 << 28), (torch.int32, 1 << 28), (torch.int64, 1 << 24)):
    x = torch.zeros(n, dtype=dt, device="cuda")
    line = []
    for mode in (0, 1):
        lib.ps_set_tuning(b"add_chunked", mode)
        for _ in range(3):
            dev.add_offset(x, 1)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            dev.add_offset(x, 1)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / 20
        line.append(f"chunked={mode}: {ms * 1e3:.1f} us {2 * n * x.element_size() / ms / 1e6:.0f} GB/s")
    assert int(x[n // 2].item()) == 46 and int(x[-1].item()) == 46
    lib.ps_set_tuning(b"add_chunked", 1)
    print(dt, n, "  ".join(line), flush=True)
