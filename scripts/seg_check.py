"""Correctness of a library build on CSR segments (numpy reference): python scripts/seg_check.py lib.so"""
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
r = np.random.default_rng(5)
bad = 0
for n, nseg, dt, excl in ((1 << 24, 1 << 10, np.int32, False), (1 << 24, 1 << 16, np.int32, True),
                          (1 << 24, 1 << 21, np.int32, False), ((1 << 24) + 12345, 1 << 18, np.int64, False),
                          (1 << 23, 1 << 22, np.uint32, True), (1 << 24, 77, np.int32, True)):
    x = r.integers(0, 1000, n).astype(dt)
    cuts = np.sort(r.integers(0, n + 1, nseg - 1))  # repeated offsets (empty segments) included
    offs = np.concatenate([[0], cuts, [n]]).astype(np.int64)
    acc = np.uint64 if dt == np.uint32 else np.int64
    cs = np.concatenate([[0], np.cumsum(x.astype(acc))]).astype(acc)
    seg_of = np.searchsorted(offs, np.arange(n), side="right") - 1
    want = (cs[1:] if not excl else cs[:-1]) - cs[offs[seg_of]]
    want_tot = cs[offs[1:]] - cs[offs[:-1]]
    xt = torch.from_numpy(x.view(np.int32) if dt == np.uint32 else x).cuda()
    if dt == np.uint32:
        xt = xt.view(torch.uint32)
    out = torch.empty(n, dtype=torch.uint64 if dt == np.uint32 else torch.int64, device="cuda")
    tots = torch.zeros(nseg, dtype=out.dtype, device="cuda")
    device.scan_segmented(xt, torch.from_numpy(offs).cuda(), out, exclusive=excl, seg_totals=tots)
    torch.cuda.synchronize()
    got = out.cpu().numpy().view(acc)
    gt = tots.cpu().numpy().view(acc)
    ok = np.array_equal(got, want) and np.array_equal(gt, want_tot)
    bad += not ok
    print(f"{sys.argv[1].split('/')[-1]} n={n} nseg={nseg} {np.dtype(dt).name} excl={excl}: {'ok' if ok else 'MISMATCH'}", flush=True)
sys.exit(bad)
