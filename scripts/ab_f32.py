"""cfg2 (2^28 float32 BASELINE draw) through the stream kernel with the float
pair path (float_exact=0, default) and float64 per element (float_exact=1):
time per launch (CUDA events, 20 back-to-back launches) and error vs the
reference float32(cumsum(float64))."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2312_14874_b200 import _lib, device  # noqa: E402

lib = _lib.load()
x = np.random.default_rng(1).random(1 << 28, dtype=np.float32)
ref = np.cumsum(x.astype(np.float64))
t = torch.from_numpy(x).cuda()
o = torch.empty_like(t)
for fe in (0, 1, 0, 1):
    lib.ps_set_tuning(b"float_exact", fe)
    for _ in range(3):
        device.scan(t, o)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        device.scan(t, o)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 20
    got = o.cpu().numpy()
    rel = float(np.max(np.abs(got.astype(np.float64) - ref) / ref))
    print(f"float_exact={fe}: {ms*1e3:.1f} us  {2**31/ms/1e6:.0f} GB/s  frac {2**31/ms/1e6/6551:.3f}  "
          f"max_rel {rel:.2e}  bit_exact {np.array_equal(got, ref.astype(np.float32))}")
