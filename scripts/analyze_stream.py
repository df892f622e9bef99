"""Summarise gpurun_out/trace_stream_*.bin (scripts/trace_stream.cu), ns."""
import sys
import numpy as np

for name in sys.argv[1:] or ["f32", "i64"]:
    t = np.fromfile(f"gpurun_out/trace_stream_{name}.bin", dtype=np.uint64).astype(np.int64).reshape(-1, 148, 8)
    t = t[3:-3]  # steady state
    q = lambda x: " ".join(f"{np.percentile(x, p):7.0f}" for p in (10, 50, 90, 99))
    iss, land, pub, gs, ge, pre, s0, s1 = (t[:, :, i] for i in range(8))
    print(f"== {name}: regions {t.shape[0]} (p10 p50 p90 p99, ns)")
    print(" TMA issue -> landed        :", q(land - iss))
    print(" landed -> published        :", q(pub - land))
    print(" publish -> gather start    :", q(gs - pub))
    print(" gather duration            :", q(ge - gs))
    print(" gather end - last publish  :", q(ge - pub.max(axis=1)[:, None]))
    print(" last publish - first publ. :", q(pub.max(axis=1) - pub.min(axis=1)))
    print(" gather end -> carries      :", q(pre - ge))
    print(" carries - scanner data-ready:", q(pre - s0))
    print(" scanner data-ready -> done :", q(s1 - s0))
    print(" scanner done -> next issue :", q(iss[6:] - s1[:-6]))
    print(" region period (max publish):", q(np.diff(pub.max(axis=1))))
    print(" buffer cycle (issue->issue):", q(iss[6:] - iss[:-6]))
