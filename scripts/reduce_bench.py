"""scripts/reduce_bench.py -- dev tool: read bandwidth of ps_reduce (multi-GPU phase 1,
sequential_accumulate) with block tickets (reduce_blocks=1) and grid-stride shares (0)."""
import sys, torch
sys.path.insert(0, "/root/repo")
from paper_2312_14874_b200 import _lib, device as dev
lib = _lib.load()
for dt, n in ((torch.float32, 1 << 28), (torch.int64, 1 << 28), (torch.int32, 1 << 28), (torch.int64, 1 << 24)):
    x = torch.ones(n, dtype=dt, device="cuda")
    line = []
    for mode in (0, 1):
        lib.ps_set_tuning(b"reduce_blocks", mode)
        for _ in range(3): dev.reduce(x)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20): dev.reduce(x)
        e1.record(); e1.synchronize()
        ms = e0.elapsed_time(e1) / 20
        assert int(dev.reduce(x).item()) == n
        line.append(f"blocks={mode}: {ms*1e3:.1f} us {n * x.element_size() / ms / 1e6:.0f} GB/s")
    lib.ps_set_tuning(b"reduce_blocks", 1)
    print(dt, n, "  ".join(line))
