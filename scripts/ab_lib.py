"""A/B of library builds: ``python scripts/ab_lib.py <lib.so> <cfg> [reps]`` times
ps_scan on a BASELINE config's input through the given .so (CUDA events,
back-to-back launches) and checks it against numpy.  Run once per build."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2312_14874_b200 import _build  # noqa: E402

_build.LIB_PATH = sys.argv[1]
_build.up_to_date = lambda: True
from paper_2312_14874_b200 import _lib, device  # noqa: E402
import bench  # noqa: E402

cfg = bench.CONFIGS[sys.argv[2]]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
for k, v in (a.split("=") for a in sys.argv[4:]):
    _lib.load().ps_set_tuning(k.encode(), int(v))
xh = bench.host_input(cfg)
x = torch.from_numpy(xh).cuda()
o = torch.empty(x.shape, dtype={"int64": torch.int64, "float32": torch.float32}[cfg["dout"]], device="cuda")
run = (lambda: device.scan_batched(x, o)) if "rows" in cfg else (lambda: device.scan(x, o, exclusive=cfg["exclusive"]))
for _ in range(3):
    run()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(reps):
    run()
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / reps
byts = x.numel() * (x.element_size() + o.element_size())
got = o.cpu().numpy()
if cfg["din"] == "float32":
    ref = np.cumsum(xh.astype(np.float64))
    err = f"max_rel {np.max(np.abs(got - ref) / ref):.2e}"
else:
    ref = np.cumsum(xh, axis=-1, dtype=np.int64)
    if cfg["exclusive"]:
        ref = np.concatenate([[0], ref[:-1]])
    err = f"exact {np.array_equal(got, ref)}"
print(f"{sys.argv[1].split('/')[-1]} {sys.argv[2]} {' '.join(sys.argv[4:])}: {ms*1e3:.1f} us "
      f"{byts/ms/1e6:.0f} GB/s frac {byts/ms/1e6/6551:.3f} {err}", flush=True)
