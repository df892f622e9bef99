"""Host-buffer pipeline (ps_scan_host) chunk-size sweep + raw PCIe copy rates (dev tool)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2312_14874_b200 import device  # noqa: E402

n = 1 << 28
x = torch.from_numpy(np.random.default_rng(1).random(n, dtype=np.float32)).pin_memory()
y = torch.empty_like(x).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
d2 = torch.empty(n, dtype=torch.float32, device="cuda")
for name, fn in (("H2D", lambda: d.copy_(x, non_blocking=True)), ("D2H", lambda: y.copy_(d, non_blocking=True))):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    print(f"{name} alone: {5 * 4 * n / (time.perf_counter() - t) / 1e9:.1f} GB/s")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5):
    with torch.cuda.stream(s1):
        d.copy_(x, non_blocking=True)
    with torch.cuda.stream(s2):
        y.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
print(f"H2D+D2H concurrent: {5 * 4 * n / (time.perf_counter() - t) / 1e9:.1f} GB/s per direction")
for chunk_mb in (4, 8, 16, 32, 64, 128):
    ce = (chunk_mb << 20) // 4
    device.scan_host(x, y, chunk_elems=ce)
    t = time.perf_counter()
    for _ in range(5):
        device.scan_host(x, y, chunk_elems=ce)
    dt = (time.perf_counter() - t) / 5
    print(f"scan_host chunk {chunk_mb:4d} MB: {dt * 1e3:.2f} ms  {n / dt / 1e9:.2f} Gelem/s")
ref = np.cumsum(x.numpy().astype(np.float64)).astype(np.float32)
print("bit-exact:", np.array_equal(y.numpy(), ref))
