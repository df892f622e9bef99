"""Per-rank cost of the two multi-GPU schemes, measured on ONE B200 (only one
GPU is available to this project), for the cfg5 strong split (2^31 int64 over
G = 1, 2, 4, 8 ranks): every rank's program is run on its own shard size and
timed with CUDA events on the launching stream.

  single   the one-GPU single-pass scan of the shard (no exchange: the N=1 path)
  RtS      reduce-then-scan (ACCUMULATE_SCAN_EQUAL): reduce -> exchange -> seeded scan
  StF      scan-then-fixup (SCAN_INCREMENT_EQUAL), rank > 0: scan -> exchange -> add
  exchange nccl: a real NCCL all-gather of one 8-byte total on a 1-rank
                 communicator, the totals tensor of the G ranks consumed by the
                 next kernel (seed_terms / delta_terms);
           p2p:  the fused mailbox exchange with G virtual ranks emulated on
                 this GPU (the earlier ranks publish first, in rank order, as in
                 tests/test_p2p_gpu.py): publish kernel + the consuming kernel's
                 in-kernel mailbox fold.  NVLink latency of the store is not in it.

Writes a markdown table (stdout) and a JSON line per row (gpurun_out/sharded_n1.jsonl).
"""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_14874_b200 import device as dev  # noqa: E402
from paper_2312_14874_b200.distributed import MailboxExchange  # noqa: E402

N = 1 << 31
K = 10
PEAK = 6551.0


def timed(fn, reps=K):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29517")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    rows = []
    g = torch.Generator(device="cuda").manual_seed(4)
    for G in (1, 2, 4, 8):
        n = N // G
        x = torch.randint(0, 1001, (n,), generator=g, device="cuda", dtype=torch.int64)
        out = torch.empty_like(x)
        r = G - 1  # the last rank: it waits for every predecessor
        terms = torch.randint(0, 1 << 30, (max(r, 1),), device="cuda", dtype=torch.int64)[:r]
        parts = [torch.empty(1, dtype=torch.int64, device="cuda")]

        def single():
            dev.scan(x, out)

        def rts_nccl():
            t = dev.reduce(x)
            dist.all_gather(parts, t)
            dev.scan(x, out, seed_terms=terms if r else None)

        def stf_nccl():
            t = dev.scan(x, out)
            dist.all_gather(parts, t)
            if r:
                dev.add_offset(out, 0, terms)

        boxes = [torch.zeros(2 * G * 16, dtype=torch.uint8, device="cuda") for _ in range(G)]
        ex = [MailboxExchange(boxes[h], [b.data_ptr() for b in boxes], h) for h in range(G)]
        one = torch.ones(1, dtype=torch.int64, device="cuda")
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]

        def p2p(program):
            # virtual ranks 0..r-1 publish first (outside the timed window), then rank r runs
            eps = [e.next_epoch() for e in ex]
            for h in range(r):
                ex[h].publish(one, *eps[h])
            ev[0].record()
            program(eps[r])
            ev[1].record()

        def rts_p2p(ep):
            ex[r].publish(dev.reduce(x), *ep)
            dev.scan_mailbox(x, out, ex[r].slots(ep[0]), r, ep[0], timeout=ex[r].timeout)

        def stf_p2p(ep):
            t = dev.scan(x, out)
            ex[r].publish(t, *ep)
            if r:
                delta = dev.scan_mailbox(None, None, ex[r].slots(ep[0]), r, ep[0], timeout=ex[r].timeout,
                                         dtype=torch.int64)
                dev.add_offset(out, 0, delta)

        def timed_p2p(program):
            p2p(program)
            torch.cuda.synchronize()
            tot = 0.0
            for _ in range(K):
                p2p(program)
                torch.cuda.synchronize()
                tot += ev[0].elapsed_time(ev[1])
            return tot / K

        t_single = timed(single)
        res = {"G": G, "shard": n, "single_ms": t_single,
               "rts_nccl_ms": timed(rts_nccl), "stf_nccl_ms": timed(stf_nccl),
               "rts_p2p_ms": timed_p2p(rts_p2p), "stf_p2p_ms": timed_p2p(stf_p2p)}
        for e in ex:
            e.check()
        rows.append(res)
        del x, out
        torch.cuda.empty_cache()
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/sharded_n1.jsonl", "w") as fh:
        for r_ in rows:
            fh.write(json.dumps(r_) + "\n")
    base = rows[0]["single_ms"]
    print("| G | shard elements | single-pass (ms) | RtS nccl | RtS p2p | StF nccl | StF p2p | "
          "strong speedup RtS p2p vs 1-GPU single pass | StF p2p |")
    print("|---|---|---|---|---|---|---|---|---|")
    for r_ in rows:
        print(f"| {r_['G']} | {r_['shard']} | {r_['single_ms']:.3f} | {r_['rts_nccl_ms']:.3f} | "
              f"{r_['rts_p2p_ms']:.3f} | {r_['stf_nccl_ms']:.3f} | {r_['stf_p2p_ms']:.3f} | "
              f"{base / r_['rts_p2p_ms']:.2f} | {base / r_['stf_p2p_ms']:.2f} |")
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
