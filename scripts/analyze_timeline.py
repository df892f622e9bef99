"""Per-region timeline (median/max over CTAs, us from the first TMA issue) of a
scripts/trace_stream.cu capture: python scripts/analyze_timeline.py <file.bin> [rows]"""
import sys

import numpy as np

t = np.fromfile(sys.argv[1], dtype=np.uint64).astype(np.int64).reshape(-1, 148, 8)
rows = int(sys.argv[2]) if len(sys.argv) > 2 else t.shape[0]
t = t - t[0, :, 0].min()
names = ["issue", "land", "pub", "gs", "ge", "pre", "s0", "s1"]
print("reg " + " ".join(f"{n:>13s}" for n in names))
for r in list(range(min(rows, t.shape[0]))) + list(range(max(rows, t.shape[0] - 3), t.shape[0])):
    print(f"{r:3d} " + " ".join(f"{np.median(t[r, :, i]) / 1e3:6.2f}/{t[r, :, i].max() / 1e3:6.2f}" for i in range(8)))
