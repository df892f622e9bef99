"""Locate wrong outputs of the rounds kernel at full size (development tool)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2312_14874_b200 import _lib, device  # noqa: E402

lib = _lib.load()
n = 1 << 28
flags = np.random.default_rng(2).integers(0, 2, n, dtype=np.int32)
ref = np.cumsum(flags, dtype=np.int64)
x = torch.from_numpy(flags).cuda()
for trial in range(4):
    out = torch.empty(n, dtype=torch.int64, device="cuda")
    tot = device.scan(x, out)
    got = out.cpu().numpy()
    bad = np.flatnonzero(got != ref)
    print(f"trial {trial}: total {int(tot.item())} want {int(ref[-1])} bad {bad.size}")
    if bad.size:
        first = bad[0]
        d = got - ref
        jumps = np.flatnonzero(np.diff(d) != 0)[:20] + 1
        print("  first bad", first, "diff at first", d[first])
        print("  jump positions", jumps.tolist())
        print("  jump deltas", [int(d[j] - d[j - 1]) for j in jumps])
        R = 48 << 20
        G = 148
        P = (R // 12 // G) // 8192 * 8192
        for j in jumps[:10]:
            r, off = divmod(int(j), P * G)
            c, o2 = divmod(off, P)
            print(f"   pos {j}: region {r} cta {c} offset {o2} (chunk {o2 // 1024}, elem {o2 % 1024})")
