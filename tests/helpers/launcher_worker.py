"""Rank body for tests/test_bench_launcher.py: what bench.py's N>1 leg does,
on CPU processes (gloo) with the test-only oracle ops in place of the CUDA
kernels -- shard the BASELINE-style input by the EQUAL layout, scan it with
the sharded reduce-then-scan, time it, take the max over ranks, and print
one JSON line from rank 0."""
import json
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = [ROOT, os.path.dirname(HERE)]

import bench  # noqa: E402
from test_distributed import OracleOps  # noqa: E402

from paper_2312_14874_b200.distributed import ShardedScan, shard_span  # noqa: E402
from paper_2312_14874_b200.plan import SchemeId  # noqa: E402


def main():
    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    dist.init_process_group("gloo")
    n = 100_003
    x = np.random.default_rng(4).integers(0, 1001, n, dtype=np.int64)
    sp = shard_span(n, world, rank)
    lo, ln = sp.start, sp.len
    shard = torch.from_numpy(x[lo:lo + ln].copy())
    out = torch.empty_like(shard)
    scan = ShardedScan(scheme=SchemeId.ACCUMULATE_SCAN_EQUAL, ops=OracleOps())
    t0 = time.perf_counter()
    res = scan(shard, out)
    el = bench.max_over_ranks(time.perf_counter() - t0 + rank, dist, world)  # rank skews the clock
    ok = torch.tensor([int(np.array_equal(out.numpy(), np.cumsum(x)[lo:lo + ln]))])
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    if rank == 0:
        print(json.dumps({"world": world, "ok": bool(ok.item()), "total": int(res.total.item()),
                          "want_total": int(x.sum()), "max_elapsed_ge": el >= world - 1}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
