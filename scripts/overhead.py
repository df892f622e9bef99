import sys, time
import torch
sys.path.insert(0, ".")
from paper_2312_14874_b200 import device, _lib
lib = _lib.load()
for n, dt in ((1000, torch.int64), (1 << 24, torch.int64)):
    x = torch.randint(0, 100, (n,), device="cuda", dtype=dt)
    o = torch.empty_like(x)
    for _ in range(10):
        device.scan(x, o)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(200):
        device.scan(x, o)
    cpu = (time.perf_counter() - t) / 200
    torch.cuda.synchronize()
    gpu = (time.perf_counter() - t) / 200
    print(f"n={n}: cpu enqueue {cpu*1e6:.1f} us/call, wall {gpu*1e6:.1f} us/call")
