"""scripts/ab_stream.py -- dev tool: A/B timing of stream-kernel tuning knobs and
library builds at the BASELINE sizes.

python scripts/ab_stream.py [lib.so] [knob=v1,v2,...] ; K back-to-back launches
between two events per sample (as bench.py), samples alternate between settings."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2312_14874_b200 import _build  # noqa: E402

args = sys.argv[1:]
if args and args[0].endswith(".so"):
    _build.LIB_PATH = args.pop(0)
    _build.up_to_date = lambda: True
from paper_2312_14874_b200 import _lib, device  # noqa: E402

lib = _lib.load()
knob, vals = (args[0].split("=") if args else ("stream_gather_depth", "1,3"))
vals = [int(v) for v in vals.split(",")]
CASES = [("cfg1 i64 2^24", torch.int64, torch.int64, 1 << 24, False, 100),
         ("cfg2 f32 2^28", torch.float32, torch.float32, 1 << 28, False, 20),
         ("cfg3 i32->i64 2^28 ex", torch.int32, torch.int64, 1 << 28, True, 20),
         ("i64 2^27", torch.int64, torch.int64, 1 << 27, False, 20)]
ROWS = [("cfg4 16384x16384 i32->i64", torch.int32, torch.int64, (16384, 16384), False, 20),
        ("8192x32768 f32", torch.float32, torch.float32, (8192, 32768), False, 20),
        ("16384x8192 i64", torch.int64, torch.int64, (16384, 8192), False, 20),
        ("65536x3000 i32->i64", torch.int32, torch.int64, (65536, 3000), False, 20)]
if knob.startswith("rows_"):
    CASES = ROWS
print(lib.ps_set_tuning(b"scan_kernel", 3), _build.LIB_PATH)
for name, dti, dto, n, ex, K in CASES:
    x = (torch.rand(n, device="cuda") < 0.5).to(dti) if dti != torch.float32 else torch.rand(n, device="cuda")
    out = torch.empty(n, dtype=dto, device="cuda")
    if x.dim() == 2:
        device.scan = lambda x, out, exclusive=False: device.scan_batched(x, out, exclusive=exclusive)
    res = {v: [] for v in vals}
    for rep in range(4):
        for v in vals:
            assert lib.ps_set_tuning(knob.encode(), v) == 0
            for _ in range(3):
                device.scan(x, out, exclusive=ex)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(K):
                device.scan(x, out, exclusive=ex)
            b.record()
            b.synchronize()
            res[v].append(a.elapsed_time(b) / K * 1e3)
    byt = x.numel() * (x.element_size() + out.element_size())
    print(name, "  ".join(f"{knob}={v}: {min(t):7.1f} us ({byt / min(t) / 1e3 / 6551:.3f})" for v, t in res.items()),
          flush=True)
