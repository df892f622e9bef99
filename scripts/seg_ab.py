"""A/B of library builds on the CSR region kernel: python scripts/seg_ab.py lib1.so [lib2.so ...]
(2^28 int32 -> int64; 16K and 1M random segments with totals, 1M without)"""
import subprocess
import sys

code = r'''
import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2312_14874_b200 import _build
_build.LIB_PATH = sys.argv[1]; _build.up_to_date = lambda: True
from paper_2312_14874_b200 import _lib, device
lib = _lib.load(); lib.ps_set_tuning(b"seg_kernel", 2)
n = 1 << 28; r = np.random.default_rng(10)
x = torch.from_numpy(r.integers(0, 256, n, dtype=np.int32)).cuda()
out = torch.empty(n, dtype=torch.int64, device="cuda")
res = []
for nseg, wt in ((1 << 14, True), (1 << 20, True), (1 << 20, False), (1 << 24, True)):
    offs = torch.from_numpy(np.concatenate([[0], np.sort(r.integers(1, n, nseg - 1)), [n]]).astype(np.int64)).cuda()
    tots = torch.empty(nseg, dtype=torch.int64, device="cuda") if wt else None
    for _ in range(3): device.scan_segmented(x, offs, out, seg_totals=tots)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10): device.scan_segmented(x, offs, out, seg_totals=tots)
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    res.append(f"{nseg}{'' if wt else '-notot'}: {ms*1e3:.0f} us ({(n*12+nseg*16)/ms/1e6/6456:.3f})")
print(f"{sys.argv[1].split('/')[-1]:24s} " + "  ".join(res), flush=True)
'''
for rep in range(2):
    for lib in sys.argv[1:]:
        try:
            subprocess.run([sys.executable, "-c", code, lib], timeout=150)
        except subprocess.TimeoutExpired:
            print(lib, "TIMEOUT", flush=True)
