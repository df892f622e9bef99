import sys, torch
sys.path.insert(0, "/root/repo")
from paper_2312_14874_b200 import device as dev
for dt, n in ((torch.float32, 1 << 28), (torch.int64, 1 << 28), (torch.int32, 1 << 28)):
    x = torch.ones(n, dtype=dt, device="cuda")
    for _ in range(3): dev.reduce(x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): dev.reduce(x)
    e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(dt, f"{ms*1e3:.1f} us", f"{n * x.element_size() / ms / 1e6:.0f} GB/s read")
