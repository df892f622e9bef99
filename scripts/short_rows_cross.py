"""Aligned short rows: the multi-row rows kernel (rows_kernel=2) against the uniform-segment route
of launch_scan (rows_kernel=1 -> region kernel for large inputs), by row length."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2312_14874_b200 import _lib, device  # noqa: E402

lib = _lib.load()
peak = float(json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"])
REPS = 5 if len(sys.argv) < 2 or int(sys.argv[1]) >= 26 else 50
LOGN = int(sys.argv[1]) if len(sys.argv) > 1 else 28  # log2 of the batch's elements (4-byte input)
for din, dout in ((torch.int32, torch.int64), (torch.int64, torch.int64), (torch.float32, torch.float32)):
    es = 4 if din != torch.int64 else 8
    for cols in (64, 128, 256, 512, 1024, 2048, 4096):
        rows = (1 << (LOGN if es == 4 else LOGN - 1)) // cols
        x = torch.rand((rows, cols), device="cuda").to(din) if din.is_floating_point else torch.randint(0, 256, (rows, cols), dtype=din, device="cuda")
        out = torch.empty((rows, cols), dtype=dout, device="cuda")
        res = []
        for rk in (2, 1):
            lib.ps_set_tuning(b"rows_kernel", rk)
            try:
                for _ in range(2):
                    device.scan_batched(x, out)
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for _ in range(REPS):
                    device.scan_batched(x, out)
                b.record()
                torch.cuda.synchronize()
                ms = a.elapsed_time(b) / REPS
                res.append(f"{'rows' if rk == 2 else 'segm'} {ms*1e3:7.1f} us ({rows*cols*(x.element_size()+out.element_size())/ms/1e6/peak:.3f})")
            except Exception as e:  # noqa: BLE001
                res.append(f"{'rows' if rk == 2 else 'segm'} failed: {str(e)[:40]}")
        print(f"{str(din)[6:]:>8s}->{str(dout)[6:]:<8s} cols={cols:<5d} rows={rows:<8d} " + "   ".join(res), flush=True)
lib.ps_set_tuning(b"rows_kernel", 0)
