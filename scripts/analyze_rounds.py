"""Summarise gpurun_out/trace_rounds_*.bin (scripts/trace_rounds.cu)."""
import sys
import numpy as np

for name in sys.argv[1:] or ["f32", "i64", "i32"]:
    t = np.fromfile(f"gpurun_out/trace_rounds_{name}.bin", dtype=np.uint64).astype(np.int64)
    G = 148
    t = t.reshape(-1, G, 8)
    t0 = t[0, :, 0].min()
    rs, rp, lg, lp, ss, sd = (t[:, :, i] - t0 for i in range(6))
    q = lambda x: " ".join(f"{np.percentile(x, p) / 1e3:6.2f}" for p in (10, 50, 90, 99))
    print(f"== {name} regions {t.shape[0]} total {sd.max() / 1e3:.1f} us")
    print(" reducer duration            :", q(rp - rs))
    print(" reducer idle (rs(r)-rp(r-1)):", q(rs[1:] - rp[:-1]))
    print(" gather done - last publish  :", q(lg - rp.max(axis=1)[:, None]))
    print(" prefix ready - gather done  :", q(lp - lg))
    print(" scanner duration            :", q(sd - ss))
    print(" scanner idle                :", q(ss[1:] - sd[:-1]))
    print(" region period               :", q(np.diff(sd.max(axis=1))))
