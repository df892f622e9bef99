"""A bench.py-style JSON line for the CSR-segmented workload (not a BASELINE.json config, so it
is not a `bench.py --config`): 2^28 int32 -> int64, NSEG random segments, totals requested.

    python scripts/seg_line.py [--nseg 1048576] [--steps 50] [--warmup 5] [--no-totals]

value = elements/s over K back-to-back calls (pre-pass, scan and totals gather all inside),
CUDA events on the launching stream; roofline against MEASURED_PEAKS.json for the algorithmic
bytes n*(4+8) + 16*nseg; parity: every element and every total against numpy before timing;
clocks sampled with NVML during the timed region."""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2312_14874_b200 import _lib, device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--nseg", type=int, default=1 << 20)
ap.add_argument("--steps", type=int, default=50)
ap.add_argument("--warmup", type=int, default=5)
ap.add_argument("--no-totals", action="store_true")
args = ap.parse_args()
_lib.load()
n, nseg = 1 << 28, args.nseg
r = np.random.default_rng(10)
xh = r.integers(0, 256, n, dtype=np.int32)
offs = np.concatenate([[0], np.sort(r.integers(1, n, nseg - 1)), [n]]).astype(np.int64)
x = torch.from_numpy(xh).cuda()
od = torch.from_numpy(offs).cuda()
out = torch.empty(n, dtype=torch.int64, device="cuda")
tots = None if args.no_totals else torch.empty(nseg, dtype=torch.int64, device="cuda")


def step():
    device.scan_segmented(x, od, out, seg_totals=tots)


step()
torch.cuda.synchronize()
# parity against numpy: out = S - S[segment start], totals = S[end] - S[start]
c = np.concatenate([[0], np.cumsum(xh, dtype=np.int64)])
ok = True
chunk = 1 << 26
for a in range(0, n, chunk):
    b = min(n, a + chunk)
    seg_of = np.searchsorted(offs, np.arange(a, b), side="right") - 1
    ok &= bool(np.array_equal(out[a:b].cpu().numpy(), c[a + 1:b + 1] - c[offs[seg_of]]))
if tots is not None:
    ok &= bool(np.array_equal(tots.cpu().numpy(), c[offs[1:]] - c[offs[:-1]]))
if not ok:
    raise SystemExit("seg_line: GPU result differs from numpy; refusing to time it")
del c
t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
stream = torch.cuda.current_stream()
with bench.ClockSampler(0) as clocks:
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    t0.record(stream)
    for _ in range(args.steps):
        step()
    t1.record(stream)
    torch.cuda.synchronize()
ms = t0.elapsed_time(t1) / args.steps
byts = n * 12 + nseg * 16
peak, src = bench.measured_peak()
tj = os.path.join(ROOT, "profiles", "traffic.json")
traffic = json.load(open(tj)).get("seg1m", {}).get("dram_bytes_per_launch") if nseg == 1 << 20 and os.path.exists(tj) else None
print(json.dumps({
    "metric": bench.METRIC, "value": n / (ms / 1e3), "unit": "elements/s", "n_gpus": 1, "steps": args.steps,
    "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
    "dtype": "int64", "data": "synthetic: np.random.default_rng(10) int32 uniform[0,255], random sorted cut points",
    "config": {"workload": f"CSR-segmented inclusive scan, n=2^28 int32 -> int64, {nseg} segments"
                           f"{'' if tots is None else ', segment totals'} (ps_scan_segmented)",
               "elements": n, "segments": nseg, "gpus": 1},
    "roofline": {"bound": "hbm", "achieved": byts / ms / 1e6, "peak": peak, "unit": "GB/s", "frac": byts / ms / 1e6 / peak,
                 "traffic": traffic, "peak_source": src,
                 "kernel": "seg_stream_kernel (+ seg_prepare_kernel, seg_totals_gather_kernel in the step)",
                 "kernel_avg_ms": ms, "algorithmic_bytes_per_launch": byts},
    "clocks": clocks.summary(), "gpu_launches": (3 if tots is not None else 2) * args.steps,
    "parity": {"checked": "every element and every segment total vs numpy (cumsum differences, int64)",
               "bit_exact": True, "ok": True},
}), flush=True)
