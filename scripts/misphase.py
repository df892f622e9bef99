"""1-D scans whose input and output sit at different 32-byte phases (the stream kernel's
output-aligned grid: TMA where the input's 16-byte phase fits, producer-warp copy otherwise):
correctness against numpy for every element offset pair, and timing against the look-back route."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
if len(sys.argv) > 1 and sys.argv[1].endswith(".so"):  # a variant build
    from paper_2312_14874_b200 import _build  # noqa: E402
    _build.LIB_PATH = sys.argv[1]
    _build.up_to_date = lambda: True
from paper_2312_14874_b200 import _lib, device  # noqa: E402

lib = _lib.load()
peak = float(json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"])
r = np.random.default_rng(7)
bad = 0
for din, dout in ((np.int32, np.int64), (np.int64, np.int64), (np.float32, np.float32), (np.int32, np.int32),
                  (np.float32, np.float64), (np.uint32, np.uint64)):
    n = (9 << 20) + 12345 if np.dtype(din).itemsize == 4 else (5 << 20) + 777
    fl = np.dtype(din).kind == "f"
    acc = np.float64 if fl else (np.uint64 if np.dtype(din).kind == "u" else np.int64)
    pad = 16
    xh = ((r.integers(0, 1024, n + pad) / 1024.0).astype(din) if fl else r.integers(0, 200, n + pad).astype(din))
    xd = torch.from_numpy(xh.view(np.int32) if din == np.uint32 else xh).cuda()
    if din == np.uint32:
        xd = xd.view(torch.uint32)
    tout = getattr(torch, np.dtype(dout).name)
    od = torch.empty(n + pad, dtype=tout, device="cuda")
    for oi in range(0, 8):
        for oo in range(0, 8, 1 if oi < 3 else 3):
            excl = bool((oi + oo) & 1)
            seed = 5 if oi == 2 else 0
            x = xd[oi:oi + n]
            o = od[oo:oo + n]
            o.zero_()
            tot = device.scan(x, o, exclusive=excl, seed=seed)
            c = np.cumsum(xh[oi:oi + n].astype(acc)) + acc(seed)
            want = (np.concatenate([[acc(seed)], c[:-1]]) if excl else c).astype(dout)
            got = o.cpu().numpy()
            if dout in (np.uint64, np.uint32):
                got = got.view(dout)
            tv = tot.cpu().numpy().view(acc)[0] if hasattr(tot, "cpu") else tot
            if not (np.array_equal(got, want) and tv == c[-1]):
                bad += 1
                print(f"MISMATCH {np.dtype(din).name}->{np.dtype(dout).name} in+{oi} out+{oo} excl={excl}", flush=True)
    print(f"{np.dtype(din).name}->{np.dtype(dout).name}: offsets checked, bad so far {bad}", flush=True)
# timing: 2^26 int64 with out offset +1 only, and int32->int64 with in offset +1
for din, dout, n, oi, oo in ((torch.int64, torch.int64, 1 << 26, 0, 1), (torch.int32, torch.int64, 1 << 27, 1, 0),
                             (torch.float32, torch.float32, 1 << 27, 3, 0), (torch.int32, torch.int64, 1 << 27, 2, 1)):
    x = (torch.rand(n + 8, device="cuda").to(din) if din.is_floating_point else torch.randint(0, 100, (n + 8,), dtype=din, device="cuda"))[oi:oi + n]
    o = torch.empty(n + 8, dtype=dout, device="cuda")[oo:oo + n]
    for knob in (1, 0):
        lib.ps_set_tuning(b"stream_copy_in", knob)
        for _ in range(3):
            device.scan(x, o)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            device.scan(x, o)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 10
        byts = n * (x.element_size() + o.element_size())
        print(f"{str(din)[6:]}->{str(dout)[6:]} n=2^{n.bit_length()-1} in+{oi} out+{oo} {'stream (output grid)' if knob else 'look-back tiles    '}: "
              f"{ms*1e3:7.1f} us {byts/ms/1e6:6.0f} GB/s frac {byts/ms/1e6/peak:.3f}", flush=True)
lib.ps_set_tuning(b"stream_copy_in", 1)
sys.exit(1 if bad else 0)
