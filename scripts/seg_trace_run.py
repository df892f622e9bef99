"""Run the CSR region kernel once through a PS_SEG_TRACE build (writes gpurun_out/seg_trace.bin)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2312_14874_b200 import _build  # noqa: E402
_build.LIB_PATH = sys.argv[1]
_build.up_to_date = lambda: True
from paper_2312_14874_b200 import _lib, device  # noqa: E402

lib = _lib.load()
lib.ps_set_tuning(b"seg_kernel", 2)
n, nseg = 1 << 28, int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 20
r = np.random.default_rng(10)
x = torch.from_numpy(r.integers(0, 256, n, dtype=np.int32)).cuda()
offs = torch.from_numpy(np.concatenate([[0], np.sort(r.integers(1, n, nseg - 1)), [n]]).astype(np.int64)).cuda()
out = torch.empty(n, dtype=torch.int64, device="cuda")
tots = torch.empty(nseg, dtype=torch.int64, device="cuda") if "notot" not in sys.argv else None
for _ in range(3):
    device.scan_segmented(x, offs, out, seg_totals=tots)
torch.cuda.synchronize()
