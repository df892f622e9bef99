"""One CSR-segmented scan (2^28 int32 -> int64, 2^20 segments) for profiling:
    python scripts/seg_once.py [kernel] [reps] [nseg]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2312_14874_b200 import _lib, device  # noqa: E402

lib = _lib.load()
k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
lib.ps_set_tuning(b"seg_kernel", k)
n, nseg = 1 << 28, int(sys.argv[3]) if len(sys.argv) > 3 else 1 << 20
r = np.random.default_rng(10)
x = torch.from_numpy(r.integers(0, 256, n, dtype=np.int32)).cuda()
offs = torch.from_numpy(np.concatenate([[0], np.sort(r.integers(1, n, nseg - 1)), [n]]).astype(np.int64)).cuda()
out = torch.empty(n, dtype=torch.int64, device="cuda")
tots = torch.empty(nseg, dtype=torch.int64, device="cuda")
for _ in range(reps):
    device.scan_segmented(x, offs, out, seg_totals=tots)
torch.cuda.synchronize()
print("ok", int(tots.sum().item()) == int(x.sum().item()))
