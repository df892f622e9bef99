"""scripts/select_ab.py -- dev tool: ps_select three-launch (select_kernel=1) vs single pass (2)
for byte and word flags at 2^28 elements."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2312_14874_b200 import _lib, device as dev  # noqa: E402

lib = _lib.load()
n = 1 << 28
g = torch.Generator(device="cuda").manual_seed(5)
for fdt, vdt, p in [(torch.uint8, torch.int32, 0.5), (torch.uint8, torch.int64, 0.5), (torch.uint8, torch.int32, 0.05),
                    (torch.int32, torch.int32, 0.5)]:
    f = (torch.rand(n, device="cuda", generator=g) < p).to(fdt)
    v = torch.arange(n, dtype=vdt, device="cuda")
    out = torch.empty_like(v)
    cnt = torch.empty(1, dtype=torch.int64, device="cuda")
    res = {}
    for k in (1, 2):
        lib.ps_set_tuning(b"select_kernel", k)
        for _ in range(3):
            dev.select(v, f, out, count=cnt)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            dev.select(v, f, out, count=cnt)
        b.record()
        b.synchronize()
        res[k] = a.elapsed_time(b) / 10 * 1e3
    lib.ps_set_tuning(b"select_kernel", 0)
    print(f"flags {fdt} values {vdt} p={p}: 3-launch {res[1]:.1f} us  single-pass {res[2]:.1f} us", flush=True)
