"""scripts/launch_gap.py -- dev tool: where does the time between back-to-back
stream-kernel launches go at cfg1 size (2^24 int64, ~55 us per launch)?

Compares, per step: the bench loop (events around every step), the same loop
without per-step events, the host cost of one device.scan call, and one CUDA
graph holding K scans (each with its own epoch; replayed once)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2312_14874_b200 import device  # noqa: E402


def main(n=1 << 24, dtype=torch.int64, K=50):
    x = torch.randint(0, 101, (n,), dtype=dtype, device="cuda")
    out = torch.empty_like(x)
    s = torch.cuda.current_stream()
    for _ in range(10):
        device.scan(x, out)
    torch.cuda.synchronize()

    def per_step_events():
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for k in range(K):
            ev[k][0].record(s)
            device.scan(x, out)
            ev[k][1].record(s)
        b.record(s)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / K * 1e3, sum(e0.elapsed_time(e1) for e0, e1 in ev) / K * 1e3

    def plain():
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(K):
            device.scan(x, out)
        b.record(s)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / K * 1e3

    def host_cost():
        # queue ahead behind a long sleep kernel so the host never waits for the GPU
        torch.cuda._sleep(200_000_000)
        t0 = time.perf_counter()
        for _ in range(K):
            device.scan(x, out)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        return (t1 - t0) / K * 1e6

    def graph():
        g = torch.cuda.CUDAGraph()
        gs = torch.cuda.Stream()
        gs.wait_stream(s)
        with torch.cuda.stream(gs):
            device.scan(x, out)  # scratch sized before capture
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=gs):
            for _ in range(K):
                device.scan(x, out)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        g.replay()
        b.record(s)
        torch.cuda.synchronize()
        ok = torch.equal(out, torch.cumsum(x, 0))
        return a.elapsed_time(b) / K * 1e3, ok

    for rep in range(3):
        tot, inside = per_step_events()
        print(f"[{rep}] bench loop: {tot:.2f} us/step (events inside {inside:.2f})  plain loop: {plain():.2f}"
              f"  host per call: {host_cost():.1f} us")
    try:
        gt, ok = graph()
        print(f"graph of {K}: {gt:.2f} us/step, result ok={ok}")
    except Exception as e:  # noqa: BLE001
        print("graph capture failed:", type(e).__name__, e)


if __name__ == "__main__":
    main()
    main(1 << 28, torch.float32, 20)
