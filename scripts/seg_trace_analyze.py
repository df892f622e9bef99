"""Summarise gpurun_out/seg_trace.bin (a PS_SEG_TRACE build of the CSR region kernel):
steady-state medians of the hand-off intervals, per region and CTA (us)."""
import sys

import numpy as np

path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/seg_trace.bin"
raw = np.fromfile(path, dtype=np.int64)
R, G = int(raw[0]), int(raw[1])
t = raw[2:].reshape(R, G, 8).astype(np.float64)
t0 = t[t > 0].min()
t = np.where(t > 0, t - t0, np.nan) / 1e3
a, b = R // 4, 3 * R // 4


def iv(x, y, dr=0):
    d = t[a + dr:b + dr, :, y] - t[a:b, :, x]
    return f"median {np.nanmedian(d):7.2f}  p90 {np.nanpercentile(d, 90):7.2f}"


print(f"regions {R}, CTAs {G}; regions {a}..{b}")
print("  issue -> landed            ", iv(0, 1))
print("  landed -> publish (reduce) ", iv(1, 2))
print("  ledger start -> gathered   ", iv(3, 4))
print("  gathered -> pre (fold)     ", iv(4, 5))
print("  scan_done(r-1)->prescanned(r)", iv(7, 6, 1))
print("  prescanned -> scan_done    ", iv(6, 7))
print("  pre -> scan_done           ", iv(5, 7))
print("  scan_done(r) -> issue(r+NB)", iv(7, 0, 6))
print("  issue(r) -> issue(r+1)     ", iv(0, 0, 1))
print("  ledger: pre(r) -> start(r+1)", iv(5, 3, 1))
lp, fp = np.nanmax(t[a:b, :, 2], axis=1), np.nanmin(t[a:b, :, 2], axis=1)
print(f"  publish spread within a region: {np.nanmedian(lp - fp):.2f}")
print(f"  last publish -> max gathered: {np.nanmedian(np.nanmax(t[a:b, :, 4], axis=1) - lp):.2f}")
print(f"  region period: {np.nanmedian(np.diff(np.nanmedian(t[:, :, 5], axis=1))):.2f}")
