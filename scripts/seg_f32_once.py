"""One float32 CSR-segmented scan (2^28, nseg segments) for profiling: python scripts/seg_f32_once.py [nseg] [reps]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2312_14874_b200 import _lib, device  # noqa: E402

lib = _lib.load()
lib.ps_set_tuning(b"seg_kernel", 2)
nseg = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 14
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
n = 1 << 28
r = np.random.default_rng(10)
x = torch.rand(n, dtype=torch.float32, device="cuda")
offs = torch.from_numpy(np.concatenate([[0], np.sort(r.integers(1, n, nseg - 1)), [n]]).astype(np.int64)).cuda()
out = torch.empty(n, dtype=torch.float32, device="cuda")
tots = torch.empty(nseg, dtype=torch.float64, device="cuda")
for _ in range(reps):
    device.scan_segmented(x, offs, out, seg_totals=tots)
torch.cuda.synchronize()
print("ok")
