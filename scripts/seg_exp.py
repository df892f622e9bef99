"""Timing experiments on the CSR region kernel: with/without totals, by segment count."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2312_14874_b200 import _build  # noqa: E402
if len(sys.argv) > 1:
    _build.LIB_PATH = sys.argv[1]
    _build.up_to_date = lambda: True
from paper_2312_14874_b200 import _lib, device  # noqa: E402

lib = _lib.load()
lib.ps_set_tuning(b"seg_kernel", 2)
n = 1 << 28
r = np.random.default_rng(10)
x = torch.from_numpy(r.integers(0, 256, n, dtype=np.int32)).cuda()
out = torch.empty(n, dtype=torch.int64, device="cuda")
for nseg in (1, 1 << 10, 1 << 20):
    offs = torch.from_numpy(np.concatenate([[0], np.sort(r.integers(1, n, nseg - 1)), [n]]).astype(np.int64)).cuda()
    for with_tot in (False, True):
        tots = torch.empty(nseg, dtype=torch.int64, device="cuda") if with_tot else None
        for _ in range(2):
            device.scan_segmented(x, offs, out, seg_totals=tots)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            device.scan_segmented(x, offs, out, seg_totals=tots)
        b.record()
        torch.cuda.synchronize()
        print(f"{sys.argv[1:] or ['default']} nseg={nseg} totals={with_tot}: {a.elapsed_time(b)/5*1e3:.1f} us", flush=True)
