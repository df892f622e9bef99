"""Host-side costs behind the pageable e2e path: page-locking throughput
(ps_host_register / unregister) by range size, and the e2e rate of
core.scan_into on pageable vs page-locked 2^30-element int64 arrays."""
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2312_14874_b200 as ps  # noqa: E402
from paper_2312_14874_b200 import _lib, device  # noqa: E402

lib = _lib.load()
torch.cuda.init()
n = 1 << 30
a = np.ones(n, np.int64)
b = np.zeros(n, np.int64)
b.fill(1)
for piece in (1 << 20, 8 << 20, 32 << 20, 256 << 20, 8 << 30):
    flag = ctypes.c_int(0)
    t0 = time.perf_counter()
    off = 0
    regs = []
    while off < a.nbytes:
        sz = min(piece, a.nbytes - off)
        _lib.check(lib.ps_host_register(a.ctypes.data + off, sz, ctypes.byref(flag)), "reg")
        regs.append(a.ctypes.data + off)
        off += sz
    t1 = time.perf_counter()
    for p in regs:
        lib.ps_host_unregister(p)
    t2 = time.perf_counter()
    print(f"register {a.nbytes/2**30:.0f} GiB in {piece>>20} MiB pieces: {a.nbytes/(t1-t0)/1e9:.1f} GB/s, "
          f"unregister {a.nbytes/(t2-t1)/1e9:.1f} GB/s")
for label, ctx in (("pageable", None), ("pinned", (a, b))):
    import contextlib
    cm = device.pinned_host(*ctx) if ctx else contextlib.nullcontext()
    with cm:
        ps.core.scan_into(a, b, ps.full_span(a), 0)
        t0 = time.perf_counter()
        for _ in range(3):
            ps.core.scan_into(a, b, ps.full_span(a), 0)
        dt = (time.perf_counter() - t0) / 3
    assert b[-1] == n
    print(f"e2e {label}: {n/dt/1e9:.2f} G elem/s ({2*a.nbytes/dt/1e9:.1f} GB/s both directions)")
t0 = time.perf_counter()
np.copyto(b, a)
print(f"single-thread numpy copy: {a.nbytes/(time.perf_counter()-t0)/1e9:.1f} GB/s")
