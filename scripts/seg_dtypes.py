"""CSR region kernel by dtype pair: 2^28 (4-byte) / 2^27 (8-byte) elements, 16K and 1M random
segments with totals; time per call and fraction of the measured HBM peak."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
if len(sys.argv) > 1:  # a variant build (scripts/build_variants.sh)
    from paper_2312_14874_b200 import _build  # noqa: E402
    _build.LIB_PATH = sys.argv[1]
    _build.up_to_date = lambda: True
from paper_2312_14874_b200 import _lib, device  # noqa: E402

lib = _lib.load()
lib.ps_set_tuning(b"seg_kernel", 2)
peak = float(json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"])
r = np.random.default_rng(11)
PAIRS = ((torch.int32, torch.int64), (torch.int64, torch.int64), (torch.float32, torch.float32),
         (torch.float64, torch.float64), (torch.int32, torch.int32))
if "ints" in sys.argv:
    PAIRS = PAIRS[:2]
for tin, tout in PAIRS:
    n = 1 << (28 if tin in (torch.int32, torch.float32) else 27)
    if tin.is_floating_point:
        x = torch.rand(n, dtype=tin, device="cuda")
    else:
        x = torch.randint(0, 256, (n,), dtype=tin, device="cuda")
    out = torch.empty(n, dtype=tout, device="cuda")
    acc = torch.float64 if tin.is_floating_point else torch.int64
    for nseg in (1 << 14, 1 << 20):
        offs = torch.from_numpy(np.concatenate([[0], np.sort(r.integers(1, n, nseg - 1)), [n]]).astype(np.int64)).cuda()
        tots = torch.empty(nseg, dtype=acc, device="cuda")
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
        byts = n * (x.element_size() + out.element_size()) + nseg * 16
        ok = abs(float(tots.sum().item()) - float(x.sum(dtype=acc).item())) <= 1e-9 * abs(float(tots.sum().item()))
        print(f"{str(tin)[6:]:>8s}->{str(tout)[6:]:<8s} nseg={nseg:>8d}: {ms*1e3:7.1f} us {byts/ms/1e6:6.0f} GB/s "
              f"frac {byts/ms/1e6/peak:.3f} totals-sum {'ok' if ok else 'BAD'}", flush=True)
