"""Locate wrong outputs of the rounds kernel with small regions (development tool)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2312_14874_b200 import _lib, device  # noqa: E402

lib = _lib.load()
lib.ps_set_tuning(b"scan_kernel", 2)
lib.ps_set_tuning(b"round_bytes", 1 << 20)
r = np.random.default_rng(21)
for n in (1_000_003, 5_000_011):
    x = r.integers(-1000, 1001, n, dtype=np.int64)
    ref = np.cumsum(x)
    t = torch.from_numpy(x).cuda()
    for trial in range(4):
        o = torch.empty_like(t)
        device.scan(t, o)
        got = o.cpu().numpy()
        d = got - ref
        bad = np.flatnonzero(d)
        print(f"n={n} trial {trial}: bad {bad.size}")
        if bad.size:
            jumps = np.flatnonzero(np.diff(d) != 0) + 1
            P = 4096
            G = 148
            for j in ([bad[0]] + jumps[:8].tolist()):
                rr, off = divmod(int(j), P * G)
                c, o2 = divmod(off, P)
                print(f"   pos {j}: delta {d[j]} region {rr} cta {c} offset {o2} chunk {o2 // 512} elem {o2 % 512}")
