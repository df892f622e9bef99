"""Exercise every kernel family once at small sizes against numpy (dev tool): a
quick all-kernels smoke, and the driver for compute-sanitizer runs where the
tool is available (memcheck / racecheck / synccheck):

    compute-sanitizer --tool memcheck python scripts/sanitize_smoke.py

(On this pool compute-sanitizer is closed; the parity suite's small cases,
tile-boundary sizes, unaligned views and stall injection are the substitute.)
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2312_14874_b200 import _lib, device as dev  # noqa: E402

lib = _lib.load()


def check(got, want, what):
    if not np.array_equal(got, want):
        raise SystemExit(f"MISMATCH {what}")


r = np.random.default_rng(1)
a64 = r.integers(0, 100, 3_000_017, dtype=np.int64)
a32 = r.integers(0, 100, 3_000_017, dtype=np.int32)
f32 = r.random(3_000_017, dtype=np.float32)
for k in (1, 2, 3):  # look-back, L2 rounds, stream (forced at a small size)
    lib.ps_set_tuning(b"scan_kernel", k)
    x = torch.from_numpy(a64).cuda()
    o = torch.empty_like(x)
    dev.scan(x, o)
    check(o.cpu().numpy(), np.cumsum(a64), f"scan int64 kernel {k}")
    x = torch.from_numpy(a32).cuda()
    o = torch.empty(x.shape, dtype=torch.int64, device="cuda")
    dev.scan(x, o, exclusive=True)
    check(o.cpu().numpy(), np.concatenate([[0], np.cumsum(a32, dtype=np.int64)[:-1]]), f"scan int32 excl {k}")
    x = torch.from_numpy(f32).cuda()
    dev.scan(x, torch.empty_like(x))
lib.ps_set_tuning(b"scan_kernel", 0)
rows = r.integers(0, 255, (600, 3000), dtype=np.int32)
for k in (1, 2):
    lib.ps_set_tuning(b"rows_kernel", k)
    x = torch.from_numpy(rows).cuda()
    o = torch.empty(x.shape, dtype=torch.int64, device="cuda")
    dev.scan_batched(x, o)
    check(o.cpu().numpy(), np.cumsum(rows, axis=1, dtype=np.int64), f"rows {k}")
lib.ps_set_tuning(b"rows_kernel", 0)
for shape in ((5000, 1000), (3000, 1001), (700, 250), (300, 20_001)):  # short rows, unaligned rows, uniform segments
    b = r.integers(0, 255, shape, dtype=np.int32)
    o = torch.empty(shape, dtype=torch.int64, device="cuda")
    dev.scan_batched(torch.from_numpy(b).cuda(), o)
    check(o.cpu().numpy(), np.cumsum(b, axis=1, dtype=np.int64), f"rows {shape}")
x = torch.from_numpy(a64).cuda()
check(int(dev.reduce(x).item()), int(a64.sum()), "reduce")
dev.add_offset(x, 5)
dev.shift_right(x)
flags = torch.from_numpy((r.random(3_000_017) < 0.5).astype(np.int32)).cuda()
vals = torch.from_numpy(a32).cuda()
for k in (1, 2):
    lib.ps_set_tuning(b"select_kernel", k)
    out, cnt = dev.select(vals, flags)
    check(out[:int(cnt.item())].cpu().numpy(), a32[flags.cpu().numpy() != 0], f"select {k}")
lib.ps_set_tuning(b"select_kernel", 0)
dev.select(vals, flags, partition=True)
t = torch.from_numpy(a64[: 1 << 16].copy()).cuda()
root = dev.tree_up_sweep(t)
dev.tree_down_sweep(t)
check(t.cpu().numpy(), np.concatenate([[0], np.cumsum(a64[: 1 << 16])[:-1]]), "tree sweeps")
offs = torch.tensor([0, 5, 100, 1000, 3_000_017], dtype=torch.int64, device="cuda")
dev.scan_segmented(torch.from_numpy(a64).cuda(), offs)
cuts = np.sort(r.integers(0, 3_000_018, 200_000))
offs2 = torch.from_numpy(np.concatenate([[0], cuts, [3_000_017]]).astype(np.int64)).cuda()
dev.scan_segmented(torch.from_numpy(a64).cuda(), offs2)
torch.cuda.synchronize()
print("sanitize smoke ok")
