"""CSR-segmented scans, 2^28 int32 -> int64 with random cut points, by segment
count and kernel (seg_kernel 1 = look-back tiles, 2 = shared-memory regions):
time per call (CUDA events, back-to-back, pre-pass included) and the fraction
of the measured HBM peak for the algorithmic bytes n*(4+8) + offsets + totals."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2312_14874_b200 import _lib, device  # noqa: E402

lib = _lib.load()
peak = float(json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"]) if len(sys.argv) < 2 else float(sys.argv[1])
n = 1 << 28
r = np.random.default_rng(10)
x = torch.from_numpy(r.integers(0, 256, n, dtype=np.int32)).cuda()
out = torch.empty(n, dtype=torch.int64, device="cuda")
for nseg in (1 << 14, 1 << 20, 1 << 24):
    offs = torch.from_numpy(np.concatenate([[0], np.sort(r.integers(1, n, nseg - 1)), [n]]).astype(np.int64)).cuda()
    tots = torch.empty(nseg, dtype=torch.int64, device="cuda")
    for k in (1, 2):
        lib.ps_set_tuning(b"seg_kernel", k)
        for _ in range(3):
            device.scan_segmented(x, offs, out, seg_totals=tots)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            device.scan_segmented(x, offs, out, seg_totals=tots)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 10
        byts = n * 12 + (nseg + 1) * 8 + nseg * 8
        print(f"nseg={nseg:>9d} kernel={k}: {ms*1e3:8.1f} us  {byts/ms/1e6:6.0f} GB/s  frac {byts/ms/1e6/peak:.3f}",
              flush=True)
