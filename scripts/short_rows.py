"""Short contiguous rows through ps_scan_batched (the uniform-segment route): correctness against
numpy and HBM fraction, region kernel (auto) vs look-back tiles (seg_kernel=1)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2312_14874_b200 import _lib, device  # noqa: E402

lib = _lib.load()
peak = float(json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"])
r = np.random.default_rng(3)
for rows, cols, din, dout in ((1 << 20, 250, np.int32, np.int64), (1 << 18, 1001, np.int32, np.int64),
                              (1 << 21, 127, np.int32, np.int64), (1 << 20, 250, np.float32, np.float32),
                              (1 << 19, 250, np.int64, np.int64)):
    if np.dtype(din).kind == "f":
        xh = (r.integers(0, 1024, (rows, cols)) / 1024.0).astype(din)
    else:
        xh = r.integers(0, 256, (rows, cols)).astype(din)
    x = torch.from_numpy(xh).cuda()
    out = torch.empty((rows, cols), dtype=getattr(torch, np.dtype(dout).name), device="cuda")
    acc = np.float64 if np.dtype(din).kind == "f" else np.int64
    tots = torch.empty(rows, dtype=getattr(torch, np.dtype(acc).name), device="cuda")
    want = np.cumsum(xh.astype(acc), axis=1)
    for sk in (0, 1):
        lib.ps_set_tuning(b"seg_kernel", sk)
        for excl in (False, True):
            out.zero_()
            tots.zero_()
            device.scan_batched(x, out, exclusive=excl, row_totals=tots)
            torch.cuda.synchronize()
            w = (want - xh.astype(acc)) if excl else want
            ok = np.array_equal(out.cpu().numpy(), w.astype(dout)) and np.array_equal(tots.cpu().numpy(), want[:, -1])
            if not ok:
                print(f"MISMATCH rows={rows} cols={cols} {np.dtype(din).name} seg_kernel={sk} excl={excl}", flush=True)
                sys.exit(1)
        for _ in range(2):
            device.scan_batched(x, out, row_totals=tots)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            device.scan_batched(x, out, row_totals=tots)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 10
        byts = rows * cols * (x.element_size() + out.element_size())
        print(f"{rows:>8d} x {cols:<5d} {np.dtype(din).name:>7s}->{np.dtype(dout).name:<7s} "
              f"{'region kernel' if sk == 0 else 'look-back    '}: {ms*1e3:8.1f} us {byts/ms/1e6:6.0f} GB/s frac {byts/ms/1e6/peak:.3f} ok",
              flush=True)
lib.ps_set_tuning(b"seg_kernel", 0)
