"""scripts/crossover.py -- dev tool: look-back tiles (scan_kernel=1) vs stream kernel (3)
over 1-D sizes, to place the auto threshold (rounds_min_bytes)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2312_14874_b200 import _lib, device  # noqa: E402

lib = _lib.load()
for dt, dto in ((torch.int64, torch.int64), (torch.float32, torch.float32), (torch.int32, torch.int64)):
    for lg in range(20, 27):
        n = 1 << lg
        x = torch.randint(0, 100, (n,), device="cuda").to(dt)
        o = torch.empty(n, dtype=dto, device="cuda")
        res = {}
        for k in (1, 3):
            lib.ps_set_tuning(b"scan_kernel", k)
            g = torch.cuda.CUDAGraph()  # graph of 20 launches: no host launch cost in the numbers
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                device.scan(x, o)
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=s):
                for _ in range(20):
                    device.scan(x, o)
            g.replay()
            torch.cuda.synchronize()
            best = 1e9
            for _ in range(5):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                g.replay()
                b.record()
                b.synchronize()
                best = min(best, a.elapsed_time(b) / 20 * 1e3)
            res[k] = best
        lib.ps_set_tuning(b"scan_kernel", 0)
        byt = n * (x.element_size() + o.element_size())
        print(f"{str(dt):14s} 2^{lg}: tiles {res[1]:7.1f} us ({byt / res[1] / 1e3 / 6551:.2f})  "
              f"stream {res[3]:7.1f} us ({byt / res[3] / 1e3 / 6551:.2f})  [{byt >> 20} MiB]", flush=True)
