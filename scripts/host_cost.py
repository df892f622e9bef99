"""Host cost of one device.scan call on a small input, by part (dev tool)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2312_14874_b200 import _lib, device  # noqa: E402

lib = _lib.load()
x = torch.randint(0, 100, (1 << 16,), dtype=torch.int64, device="cuda")
out = torch.empty_like(x)
tot = torch.empty(1, dtype=torch.int64, device="cuda")


def t(f, n=20000):
    for _ in range(200):
        f()
    torch.cuda.synchronize()
    a = time.perf_counter()
    for _ in range(n):
        f()
    b = time.perf_counter()
    torch.cuda.synchronize()
    return (b - a) / n * 1e6


print("device.scan(x, out)                 %.2f us" % t(lambda: device.scan(x, out), 5000))
print("device.scan(x, out, total=tot)      %.2f us" % t(lambda: device.scan(x, out, total=tot), 5000))
print("torch.empty(1, device)              %.2f us" % t(lambda: torch.empty(1, dtype=torch.int64, device=x.device)))
print("current_stream().cuda_stream        %.2f us" % t(lambda: torch.cuda.current_stream(x.device).cuda_stream))
print("is_current_stream_capturing         %.2f us" % t(torch.cuda.is_current_stream_capturing))
print("ps_scan_scratch_bytes (ctypes)      %.2f us" % t(lambda: lib.ps_scan_scratch_bytes(1 << 16, 2, 2)))
print("x.data_ptr() x2                     %.2f us" % t(lambda: (x.data_ptr(), out.data_ptr())))
print("torch.cumsum(x) for comparison      %.2f us" % t(lambda: torch.cumsum(x, 0, out=out), 5000))
