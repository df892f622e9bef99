"""Per-sub-tile scanner timeline of CTA 0 (gpurun_out/trace_sub_<name>.bin, scripts/trace_rounds.cu)."""
import sys
import numpy as np

SW = 8
for name, nsub in [(a.split(":")[0], int(a.split(":")[1])) for a in sys.argv[1:]]:
    t = np.fromfile(f"gpurun_out/trace_sub_{name}.bin", dtype=np.uint64).astype(np.int64)
    t = t.reshape(-1, nsub, SW + 1, 4)
    R = t.shape[0]
    t0 = t[0, 0, :SW, 0].min()
    sc = t[:, :, :SW, :3] - t0
    pr = t[:, :, SW, :2] - t0
    q = lambda x: " ".join(f"{np.percentile(x, p):7.0f}" for p in (10, 50, 90))
    wait = sc[..., 1] - sc[..., 0]
    work = sc[..., 2] - sc[..., 1]
    print(f"== {name}: regions {R} sub-tiles/region {nsub}  (ns, p10 p50 p90)")
    print(" scanner wait for TMA stage :", q(wait[2:]))
    print(" scanner work per chunk     :", q(work[2:]))
    print(" producer wait for empty    :", q((pr[2:, :, 1] - pr[2:, :, 0]).ravel()))
    # time from producer issue to the slowest scanner warp seeing the data
    print(" issue -> last warp ready   :", q((sc[2:, :, :, 1].max(axis=2) - pr[2:, :, 1]).ravel()))
    print(" issue -> first warp ready  :", q((sc[2:, :, :, 1].min(axis=2) - pr[2:, :, 1]).ravel()))
    r = R // 2
    print(" region", r, "warp0 timeline:", (sc[r, :, 0, :] - sc[r, 0, 0, 0]).tolist())
    print(" region", r, "producer      :", (pr[r] - sc[r, 0, 0, 0]).tolist())
