"""Benchmark of the B200 prefix-sum hot path (the driver's contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config cfg1..cfg5] [--scaling weak|strong]
                    [--scheme accumulate-scan|scan-increment] [--exchange p2p|nccl]

One JSON line on rank 0.  A "step" is one pass of the hot path over one batch
of the config's synthetic input.  The default workload is cfg5 (BASELINE.json
configs[4], n = 2^31 int64 uniform [0, 1000], seed 4): the config the metric
("... at 1/2/4/8 GPUs") is quoted on and the largest that fits one GPU.  The
other configs are extra lines (``--config cfgN``).

Inputs.  At N=1 (and for rank 0's shard at N>1, weak scaling) the input is the
exact BASELINE generator on the host (``np.random.default_rng(seed)...``),
copied to HBM before timing.  Strong scaling at N>1 splits that same host draw
by the EQUAL layout (rank 0 generates it once and sends every rank its shard
over NCCL).  Weak scaling at N>1 gives ranks 1..N-1 device draws of the same
distribution (``torch.randint`` / ``torch.rand``); the ``data`` field says so.

value     elements/s of the whole job, inputs resident in HBM, CUDA events on
          the launching stream, max over ranks.  Every config moves >= 256 MB
          per step against the 126 MB L2 (cfg1 is the only one of the same
          order; its in+out is 2.1x L2, stated in ``setup.l2``).
e2e       the same metric through the public drop-in API
          (``paper_2312_14874_b200.core.scan_into`` / ``device.scan_batched_host``)
          on HOST buffers, H2D + scan + D2H inside the timed region, with the
          buffers page-locked (``device.pinned_host``); ``e2e_pageable`` is the
          same call on the plain numpy arrays the reference's users pass.
roofline  the scan kernel's algorithmic bytes n * (sizeof in + sizeof out) over
          its average launch time vs the measured HBM copy peak
          (MEASURED_PEAKS.json).
cpu_baseline / --impl reference
          the reference's CPU algorithm (engine.py two-pass schemes, the
          paper's P-variants of bench.py:29-43 restated in C in oracle/) on
          every host core: SIMD2-P (the paper's recommendation) is always
          reported, ``value`` is the best of {SIMD1-P, SIMD2-P, Scalar1-P,
          Scalar2-P} on the full workload.

N>1: launched by torchrun (RANK/WORLD_SIZE in the environment) -- or, when
``--gpus N`` is given without it, bench.py re-executes itself under
``torch.distributed.run`` with N local ranks.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "scan elements/s and achieved HBM GB/s (% of B200 peak) at 1/2/4/8 GPUs vs CPU ref"
NOMINAL_HBM_GBS = 8000.0

CONFIGS = {
    "cfg1": dict(desc="cfg1: inclusive scan, n=2^24 int64 uniform[0,100] seed 0 -> int64", n=1 << 24,
                 din="int64", dout="int64", exclusive=False, seed=0, lo=0, hi=101),
    "cfg2": dict(desc="cfg2: inclusive scan, n=2^28 float32 uniform[0,1) seed 1 -> float32", n=1 << 28,
                 din="float32", dout="float32", exclusive=False, seed=1),
    "cfg3": dict(desc="cfg3: exclusive scan (partition offsets), n=2^28 int32 Bernoulli(0.5) flags seed 2 -> int64",
                 n=1 << 28, din="int32", dout="int64", exclusive=True, seed=2, lo=0, hi=2),
    "cfg4": dict(desc="cfg4: batched delta decoding, 16384 rows x 16384 int32 uniform[0,255] seed 3 -> int64 per row",
                 n=1 << 28, rows=16384, cols=16384, din="int32", dout="int64", exclusive=False, seed=3, lo=0, hi=256),
    "cfg5": dict(desc="cfg5: large scan, n=2^31 int64 uniform[0,1000] seed 4 -> int64", n=1 << 31,
                 din="int64", dout="int64", exclusive=False, seed=4, lo=0, hi=1001),
}
# the reference engine's total on the exact cfg5 input (re-checked on the GPU box host)
KNOWN_TOTALS = {"cfg5": 1073746006907}
ARITH = {"int64": "int64", "int32": "int64", "float32": "f64", "uint32": "uint64"}


def host_input(cfg, n=None):
    """The exact BASELINE.json generator, numpy PCG64."""
    n = cfg["n"] if n is None else n
    rng = np.random.default_rng(cfg["seed"])
    if cfg["din"] == "float32":
        return rng.random(n, dtype=np.float32)
    shape = (cfg["rows"], n // cfg["rows"]) if "rows" in cfg else n
    return rng.integers(cfg["lo"], cfg["hi"], shape, dtype=np.dtype(cfg["din"]))


def cpu_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def bench_config(cfg, gpus: int, scaling: str) -> dict:
    """The workload description both arms print (identical by construction)."""
    if "rows" in cfg:
        rows_per = cfg["rows"] if scaling == "weak" else math.ceil(cfg["rows"] / gpus)
        per = rows_per * cfg["cols"]
    else:
        per = cfg["n"] if scaling == "weak" else math.ceil(cfg["n"] / gpus)
    total = cfg["n"] * gpus if scaling == "weak" else cfg["n"]
    return {"workload": cfg["desc"], "elements": total, "elements_per_gpu": per, "gpus": gpus,
            "scaling": scaling}


# ---- CPU legs: the reference's algorithm restated in C (oracle/) -------------------------------

# bench.py:29-43 of the reference: label -> (engine scheme, lane width); the partitioned (-P)
# variants run with block_len = default_block_len() (plan.py:331-346)
P_SCHEMES = {"SIMD2-P": ("accumulate-scan+1", 16), "SIMD1-P": ("scan-increment+1", 16),
             "Scalar2-P": ("accumulate-scan+1", 0), "Scalar1-P": ("scan-increment+1", 0)}
# cfg4 has no engine entry point: per-row horizontal_scan (SIMD) or scalar scans on all cores
ROW_SCHEMES = {"SIMD rows": 16, "Scalar rows": 0}


class CpuPath:
    """One config's CPU path with every label it can run; ``run`` returns seconds."""

    def __init__(self, cfg, x: np.ndarray, out: np.ndarray, cores: int):
        from oracle import oracle  # the checker / CPU baseline: never on the GPU path
        from paper_2312_14874_b200.plan import default_block_len

        self.o, self.cfg, self.x, self.out, self.cores = oracle, cfg, x, out, cores
        self.block = default_block_len()
        self.rows = "rows" in cfg
        self.labels = list(ROW_SCHEMES) if self.rows else list(P_SCHEMES)
        self.paper_label = "SIMD rows" if self.rows else "SIMD2-P"

    def run(self, label: str) -> float:
        o, x, out = self.o, self.x, self.out
        if self.rows:
            t0 = time.perf_counter()
            o.rows_scan_widen_i32_i64(x, threads=self.cores, simd_w=ROW_SCHEMES[label], out=out)
            return time.perf_counter() - t0
        scheme, w = P_SCHEMES[label]
        t0 = time.perf_counter()
        if x.dtype != out.dtype:
            np.copyto(out, x)  # no mixed-dtype entry point: the widening copy is part of the path
            o.engine_scan(out, None, threads=self.cores, scheme=scheme, block_len=self.block, simd_w=w)
        else:
            o.engine_scan(x, out, threads=self.cores, scheme=scheme, block_len=self.block, simd_w=w)
        if self.cfg["exclusive"]:
            o.exclusive_from_inclusive(out)
        return time.perf_counter() - t0


def cpu_survey(path: CpuPath, reps: int) -> dict:
    """Median seconds of every label (one untimed warm-up each)."""
    res = {}
    for lab in path.labels:
        path.run(lab)
        res[lab] = statistics.median(path.run(lab) for _ in range(reps))
    return res


def cpu_baseline(cfg, x: np.ndarray, out: np.ndarray, cores: int, reps: int = 3) -> dict:
    path = CpuPath(cfg, x, out, cores)
    med = cpu_survey(path, reps)
    best = min(med, key=med.get)
    n = x.size
    return {"value": n / med[best], "unit": "elements/s", "cores": cores, "kind": "port", "label": best,
            "paper_recommended": {"label": path.paper_label, "value": n / med[path.paper_label]},
            "schemes": {lab: n / t for lab, t in med.items()},
            "sample": (f"full workload ({n} elements), every label median of {reps} after 1 warm-up; oracle/ C "
                       f"restatement of the reference engine (engine.py:278-377) with block_len="
                       f"default_block_len()={path.block}" if not path.rows else
                       f"full workload ({n} elements), per-row scans on {cores} threads, median of {reps}")}


def run_reference(args, cfg):
    """The reference arm: the reference's CPU path on the host cores, rank 0 only."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    cores = cpu_cores()
    x = host_input(cfg)
    out = np.zeros(x.shape, np.dtype(cfg["dout"]))  # faulted in outside the timer (bench.py:188-189)
    path = CpuPath(cfg, x, out, cores)
    survey = cpu_survey(path, 1)
    best = min(survey, key=survey.get)
    for _ in range(args.warmup):
        path.run(best)
    times = [path.run(best) for _ in range(args.steps)]
    tot = sum(times)
    value = x.size * args.steps / tot
    scope = ("the whole job" if args.gpus == 1 or args.scaling == "strong"
             else f"one GPU's share (1/{args.gpus} of the job)")
    line = {"metric": METRIC, "impl": "reference", "value": value, "unit": "elements/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": ARITH[cfg["din"]],
            "data": data_label(cfg, 1, "weak", host_only=True),
            "config": bench_config(cfg, args.gpus, args.scaling),
            "cpu_baseline": {"value": value, "unit": "elements/s", "cores": cores, "kind": "port", "label": best,
                             "paper_recommended": {"label": path.paper_label,
                                                   "value": x.size / survey[path.paper_label]},
                             "schemes": {lab: x.size / t for lab, t in survey.items()},
                             "sample": f"{x.size} elements per step ({scope}), the exact BASELINE draw; label "
                                       f"chosen as the fastest of {path.labels} (one timed run each)"},
            "e2e": {"value": value, "unit": "elements/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---- clocks during the timed region --------------------------------------------------------------

REASON_BITS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}


class ClockSampler:
    def __init__(self, device_index: int, period_s: float = 0.005):
        self.samples, self.reasons = [], set()
        self.period = period_s
        self._stop = threading.Event()
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None
        self.t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            self._sample()
            time.sleep(self.period)

    def _sample(self):
        if self.nv is None:
            return
        try:
            self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            bits = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            for b, name in REASON_BITS.items():
                if bits & b:
                    self.reasons.add(name)
        except Exception:
            pass

    def __enter__(self):
        self._sample()
        self.t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self.t.join()
        self._sample()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons - {"gpu_idle"}), "samples": len(self.samples)}


# ---- multi-process plumbing -----------------------------------------------------------------------

def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def launch_ranks(nproc: int, script: str, argv: list, env_extra: dict | None = None) -> int:
    """Re-execute ``script argv`` as ``nproc`` local ranks under torch.distributed.run
    (rendezvous on 127.0.0.1); returns the launcher's exit code.  Rank 0's stdout is
    the caller's stdout, so the one JSON line passes straight through."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", script, *argv]
    env = dict(os.environ)
    env.update(env_extra or {})
    env.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.call(cmd, env=env)


def max_over_ranks(value: float, dist, world: int, device=None) -> float:
    if world == 1:
        return value
    import torch
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---- GPU leg --------------------------------------------------------------------------------------

def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def committed_traffic(config_name):
    """DRAM bytes per launch of the dominant kernel from the committed ncu
    launch list (profiles/traffic.json, written by scripts/summarize_ncu.py)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            entry = json.load(fh).get(config_name)
        return None if entry is None else float(entry["dram_bytes_per_launch"])
    except Exception:
        return None


def dominant_kernel(lib, cfg, esize_in):
    """Which kernel ps_scan / ps_scan_batched dispatches for this workload."""
    if "rows" in cfg:
        if lib.ps_get_tuning(b"rows_kernel") != 1 and cfg["rows"] >= 2 * 148:
            return "scan_rows_kernel (one CTA per row, TMA-streamed 64 KiB segments)"
        return "scan_tiles_kernel (batched rows, decoupled look-back)"
    kern = lib.ps_get_tuning(b"scan_kernel")
    big = cfg["n"] * esize_in >= lib.ps_get_tuning(b"rounds_min_bytes")
    if kern == 3 or (kern == 0 and big):
        return "scan_stream_kernel (accumulate-scan over shared-memory-resident regions)"
    if kern == 2:
        return "scan_rounds_kernel (cache-partitioned accumulate-scan over L2 regions)"
    return "scan_tiles_kernel (single-pass decoupled look-back)"


def data_label(cfg, world: int, scaling: str, host_only: bool = False) -> str:
    gen = ("np.random.default_rng(%d).random(n, float32)" % cfg["seed"] if cfg["din"] == "float32" else
           "np.random.default_rng(%d).integers(%d, %d, %s, %s)" % (
               cfg["seed"], cfg["lo"], cfg["hi"],
               f"({cfg['rows']}, {cfg['cols']})" if "rows" in cfg else "n", cfg["din"]))
    if host_only:
        return f"synthetic: the exact BASELINE.json draw {gen} in host memory"
    if world == 1:
        return f"synthetic: the exact BASELINE.json draw {gen} on the host, copied to HBM before timing"
    if scaling == "strong":
        return (f"synthetic: the exact BASELINE.json draw {gen} on rank 0's host, split by the EQUAL layout "
                f"and sent to every rank over NCCL before timing")
    return (f"synthetic: rank 0's shard is the exact BASELINE.json draw {gen}; ranks 1..{world - 1} draw the "
            f"same distribution on the device (torch generator seeded {cfg['seed']}*1000+rank)")


def _device_draw(cfg, shape, rank, dev_t):
    import torch
    g = torch.Generator(device=dev_t).manual_seed(cfg["seed"] * 1000 + rank)
    if cfg["din"] == "float32":
        return torch.rand(shape, generator=g, device=dev_t, dtype=torch.float32)
    dt = {"int64": torch.int64, "int32": torch.int32}[cfg["din"]]
    return torch.randint(cfg["lo"], cfg["hi"], shape, generator=g, device=dev_t, dtype=dt)


def make_inputs(cfg, world, rank, scaling, dev_t, dist):
    """This rank's input in HBM, plus the host array it came from (None when
    device-drawn) and the shard's [start, len) in the global array."""
    import torch
    from paper_2312_14874_b200.plan import equal_shards

    rows = cfg.get("rows")
    esize = np.dtype(cfg["din"]).itemsize
    if world == 1:
        xh = host_input(cfg)
        return torch.from_numpy(xh).to(dev_t), xh, (0, cfg["n"])
    if scaling == "weak":
        if rank == 0:
            xh = host_input(cfg)
            return torch.from_numpy(xh).to(dev_t), xh, (0, cfg["n"])
        shape = (rows, cfg["cols"]) if rows else (cfg["n"],)
        return _device_draw(cfg, shape, rank, dev_t), None, (rank * cfg["n"], cfg["n"])
    # strong: rank 0 draws the whole input once and sends every rank its EQUAL shard
    units = rows if rows else cfg["n"]
    spans = [(sp.start, sp.len) for sp in equal_shards(units, world, align=1 if rows else max(1, 32 // esize))]
    lo, ln = spans[rank]
    tdt = {"int64": torch.int64, "int32": torch.int32, "float32": torch.float32}[cfg["din"]]
    shape = (ln, cfg["cols"]) if rows else (ln,)
    if rank == 0:
        xh = host_input(cfg)
        full = torch.from_numpy(xh).to(dev_t)
        for r in range(1, world):
            a, b = spans[r]
            dist.send(full[a:a + b].contiguous(), dst=r)
        x = full[lo:lo + ln].clone()
        del full
        torch.cuda.synchronize()
        return x, xh[lo:lo + ln], (lo, ln)
    x = torch.empty(shape, dtype=tdt, device=dev_t)
    dist.recv(x, src=0)
    return x, None, (lo, ln)


def verify_host(cfg, x_host: np.ndarray, out, chunk: int = 1 << 26) -> dict:
    """Chunk-wise comparison of the device result with the reference's result on
    the same host input: np.cumsum continued with the running carry (== the
    reference below 2^53; float32 = float32(cumsum(float64)),
    the reference's own rounding).  Raises on any mismatch."""
    import torch
    fl = cfg["din"] == "float32"
    excl = cfg["exclusive"]
    if "rows" in cfg:
        step = max(1, chunk // cfg["cols"])
        for r0 in range(0, x_host.shape[0], step):
            got = out[r0:r0 + step].cpu().numpy()
            ref = np.cumsum(x_host[r0:r0 + step], axis=1, dtype=np.int64)
            if not np.array_equal(got, ref):
                raise SystemExit(f"bench: GPU rows differ from the reference in rows [{r0}, {r0 + step})")
        return {"checked": "every row bit-exact vs np.cumsum(axis=1, int64) (== per-row reference scans)",
                "bit_exact": True, "ok": True}
    n = x_host.shape[0]
    carry = 0.0 if fl else 0
    max_rel, bit = 0.0, True
    flat = out.reshape(-1)
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        got = flat[a:b].cpu().numpy()
        if fl:
            inc = np.cumsum(x_host[a:b].astype(np.float64)) + carry
            ref = np.concatenate([[carry], inc[:-1]]) if excl else inc
            rel = np.abs(got.astype(np.float64) - ref) / np.maximum(np.abs(ref), 1e-30)
            max_rel = max(max_rel, float(rel.max()))
            bit = bit and bool(np.array_equal(got, ref.astype(np.float32)))
            carry = float(inc[-1])
        else:
            inc = np.cumsum(x_host[a:b], dtype=np.int64) + carry
            ref = np.concatenate([[carry], inc[:-1]]) if excl else inc
            if not np.array_equal(got, ref):
                bad = a + int(np.flatnonzero(got != ref)[0])
                raise SystemExit(f"bench: GPU result differs from the reference at index {bad}; refusing to time it")
            carry = int(inc[-1])
        del got
    res = {"checked": f"chunk-wise vs np.cumsum with carry over all {n} elements (== the reference's output)",
           "total": carry}
    if fl:
        if max_rel > 1e-4:
            raise SystemExit(f"bench: float32 result off by {max_rel:.3e} relative (> 1e-4)")
        res.update({"max_rel_err": max_rel, "tolerance": 1e-4, "bit_exact": bit, "ok": True})
    else:
        res.update({"bit_exact": True, "ok": True})
    torch.cuda.synchronize()
    return res


def verify_sharded(cfg, x, out, dist, world, rank):
    """Size-independent checks of a sharded 1-D scan on the device: the first
    differences of this rank's output reproduce its input, and its first
    output is the exact carry (sum of every earlier rank's shard) plus its
    first input.  Integers exact, float32 within 1e-5 relative."""
    import torch
    fl = cfg["din"] == "float32"
    acc = torch.float64 if fl else torch.int64
    xs = x.to(acc)
    o = out.to(acc)
    local = xs.sum().reshape(1)
    parts = [torch.empty_like(local) for _ in range(world)]
    dist.all_gather(parts, local)
    tot = torch.cat(parts)
    carry = tot[:rank].sum() if rank else torch.zeros((), dtype=acc, device=x.device)
    diff_ref = xs[:-1] if cfg["exclusive"] else xs[1:]
    first = carry if cfg["exclusive"] else carry + xs[0]
    if fl:
        scale = torch.maximum(o[-1].abs(), torch.tensor(1e-30, dtype=acc, device=x.device))
        d_ok = float(((o[1:] - o[:-1]) - diff_ref).abs().max() / scale) <= 1e-6
        f_ok = float(((o[0] - first).abs() / torch.clamp(first.abs(), min=1e-30))) <= 1e-5
    else:
        d_ok = torch.equal(o[1:] - o[:-1], diff_ref)
        f_ok = bool((o[0] == first).item())
    last = float(o[-1].item()) if fl else int(o[-1].item())
    del xs, o
    ok = torch.tensor([1 if (d_ok and f_ok) else 0], device=x.device)
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    if not int(ok.item()):
        raise SystemExit("bench: sharded GPU result fails the carry / first-difference checks; refusing to time it")
    return {"checked": "every rank: first differences reproduce the shard, first output = exact carry "
                       "(sum of earlier shards) + first input", "ok": True, "last_rank_last_output": last}


def verify_rows_device(x, out, dist, world):
    import torch
    ok = torch.equal(torch.cumsum(x.to(torch.int64), dim=1), out)
    t = torch.tensor([1 if ok else 0], device=x.device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
    if not int(t.item()):
        raise SystemExit("bench: batched rows differ from torch.cumsum on some rank; refusing to time it")
    return {"checked": "every rank's rows bit-exact vs torch.cumsum(int64) on the device", "ok": True}


def make_sharded(scheme, exchange, world, cls=None):
    """The multi-GPU scan with the requested shard-total exchange; the fused
    peer-memory exchange falls back to the NCCL all-gather (still on the GPU)
    when the symmetric-memory rendezvous is unavailable on this box."""
    if cls is None:
        from paper_2312_14874_b200.distributed import ShardedScan as cls
    ShardedScan = cls
    if exchange == "p2p" and world > 1:
        try:
            return ShardedScan(scheme=scheme, exchange="p2p"), "p2p"
        except Exception as exc:  # noqa: BLE001 - reported in the JSON line
            print(f"bench: fused p2p exchange unavailable ({exc}); using the NCCL all-gather", file=sys.stderr)
            return ShardedScan(scheme=scheme, exchange="nccl"), f"nccl (p2p unavailable: {type(exc).__name__})"
    return ShardedScan(scheme=scheme, exchange="nccl"), "nccl" if world > 1 else "none (1 GPU)"


def run_ours(args, cfg, cfg_name):
    import torch
    import torch.distributed as dist

    from paper_2312_14874_b200 import _lib, device
    from paper_2312_14874_b200.plan import SchemeId

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev_t = torch.device("cuda", local)
    sharded_1d = (world > 1 or args.force_sharded) and "rows" not in cfg
    if world > 1 or args.force_sharded:
        if not dist.is_initialized():
            if world == 1:
                os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
                os.environ.setdefault("MASTER_PORT", str(free_port()))
                os.environ.setdefault("RANK", "0")
                os.environ.setdefault("WORLD_SIZE", "1")
            dist.init_process_group("nccl", device_id=dev_t)
    _lib.load()  # fails loudly if the sm_100a library is missing
    scaling = args.scaling
    tdt = {"int64": torch.int64, "int32": torch.int32, "float32": torch.float32}

    x, x_host, (g_lo, g_len) = make_inputs(cfg, world, rank, scaling, dev_t, dist)
    out = torch.empty(x.shape, dtype=tdt[cfg["dout"]], device=dev_t)
    stream = torch.cuda.current_stream(dev_t)
    exclusive = cfg["exclusive"]
    rows = cfg.get("rows")
    scheme = SchemeId(args.scheme)
    exchange = "none (1 GPU)"
    comm = {"backend": "nccl", "nranks": dist.get_world_size()} if dist.is_initialized() else None

    if not sharded_1d:
        def step():
            if rows:
                device.scan_batched(x, out, exclusive=exclusive)
            else:
                device.scan(x, out, exclusive=exclusive)
        launches_per_step = 1
    else:
        sharded, exchange = make_sharded(scheme, args.exchange, world)
        # rank 0 of a strong split seeds nothing; every shard continues the global order
        def step():
            sharded(x, out, exclusive=exclusive, want_total=False)
        launches_per_step = launches_sharded(scheme is SchemeId.ACCUMULATE_SCAN_EQUAL, exchange == "p2p", rank)

    # ---- verify before timing (bench.py:186-192 of the reference: never time a wrong result) ----
    if world > 1:
        torch.cuda.synchronize()
        dist.barrier()
    step()
    torch.cuda.synchronize()
    if world == 1 and x_host is not None and not sharded_1d:
        parity = verify_host(cfg, x_host, out)
        if cfg_name in KNOWN_TOTALS and parity["total"] != KNOWN_TOTALS[cfg_name]:
            raise SystemExit(f"bench: total {parity['total']} != the reference's {KNOWN_TOTALS[cfg_name]}")
        if cfg_name in KNOWN_TOTALS:
            parity["reference_total"] = KNOWN_TOTALS[cfg_name]
    elif rows:
        parity = verify_rows_device(x, out, dist, world)
    else:
        parity = verify_sharded(cfg, x, out, dist, world, rank)
        if scaling == "strong" and cfg_name in KNOWN_TOTALS:
            want = KNOWN_TOTALS[cfg_name] if rank == world - 1 else None
            t = torch.tensor([0 if want is None or parity["last_rank_last_output"] == want else 1], device=dev_t)
            if world > 1:
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
            if int(t.item()):
                raise SystemExit("bench: the strong-scaled global total differs from the reference's")
            parity["reference_total"] = KNOWN_TOTALS[cfg_name]
        parity.pop("last_rank_last_output", None)

    # ---- timed region: K back-to-back steps between two events on the launching stream ----
    # (the clock sampler thread starts before the warm-up, so its start-up never delays
    # the first timed launches; it keeps sampling through the timed region)
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t_start.record(stream)
        for _ in range(args.steps):
            step()
        t_end.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    if sharded_1d and getattr(sharded, "mailbox", None) is not None:
        sharded.mailbox.check()  # a fused-exchange wait that gave up invalidates the run
    elapsed_ms = max_over_ranks(t_start.elapsed_time(t_end), dist, world, dev_t)
    job_elems = cfg["n"] * world if scaling == "weak" else cfg["n"]
    value = job_elems * args.steps / (elapsed_ms / 1e3)

    # dominant kernel = the scan.  At N=1 a step is one scan launch (launch gaps included in
    # its average); in the sharded path a scan-only loop on the same stream times it
    kernel_ms = elapsed_ms / args.steps
    if sharded_1d:
        kernel_ms = scan_kernel_ms(device, x, out, exclusive, stream, args.steps)
    n_local = x.numel()
    bytes_per_launch = n_local * (x.element_size() + out.element_size())
    achieved = bytes_per_launch / (kernel_ms / 1e3) / 1e9
    peak, peak_src = measured_peak()

    # ---- e2e through the public API on host buffers ----
    e2e = e2e_pageable = None
    if not args.no_e2e:
        e2e, e2e_pageable = measure_e2e(args, cfg, device, dist, world, rank, dev_t, x, x_host, out, scheme,
                                        sharded_1d)

    cpu = None
    if world == 1 and rank == 0 and not args.no_cpu and x_host is not None:
        out_h = np.zeros(x_host.shape, np.dtype(cfg["dout"]))
        cpu = cpu_baseline(cfg, x_host, out_h, cpu_cores())
        del out_h

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "elements/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": ARITH[cfg["din"]],
            "data": data_label(cfg, world, scaling),
            "config": bench_config(cfg, world, scaling),
            "setup": {"parallelism": (f"{world} GPU(s), contiguous EQUAL shards, {scheme.value}, exchange "
                                      f"{exchange}" if sharded_1d else
                                      f"{world} GPU(s), independent row blocks" if world > 1 else "1 GPU"),
                      "comm": comm,
                      "l2": (f"no flush: input {n_local * x.element_size() / 1e6:.0f} MB + output "
                             f"{n_local * out.element_size() / 1e6:.0f} MB per step and GPU vs 126 MB L2")},
            "achieved_gbs": achieved, "hbm_frac_measured": achieved / peak,
            "hbm_frac_nominal": achieved / NOMINAL_HBM_GBS,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": committed_traffic(cfg_name) if world == 1 else None,
                         "peak_source": peak_src,
                         "kernel": dominant_kernel(_lib.load(), cfg, x.element_size()), "kernel_avg_ms": kernel_ms,
                         "algorithmic_bytes_per_launch": bytes_per_launch},
            "cpu_baseline": cpu, "e2e": e2e, "e2e_pageable": e2e_pageable, "clocks": clocks.summary(),
            "gpu_launches": launches_per_step * args.steps, "parity": parity,
        }
        print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()


def launches_sharded(reduce_then_scan: bool, p2p: bool, rank: int) -> int:
    """Our kernels per sharded step (the NCCL all-gather is NCCL's, not counted):
    reduce-then-scan = reduce + scan (+ publish with the fused exchange, whose
    scan polls the mailbox); scan-then-fixup = scan (+ publish) and, on ranks
    > 0, the add (+ the mailbox fold that forms its delta)."""
    if reduce_then_scan:
        return 3 if p2p else 2
    return (2 + (2 if rank else 0)) if p2p else (1 + (1 if rank else 0))


def scan_kernel_ms(device, x, out, exclusive, stream, steps):
    import torch
    reps = max(5, min(steps, 50))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(reps):
        device.scan(x, out, exclusive=exclusive)
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


E2E_SAMPLE_MAX = 1 << 28  # elements per rank for the N>1 e2e (host RAM: 8 ranks x (in + out))


def measure_e2e(args, cfg, device, dist, world, rank, dev_t, x, x_host, out, scheme, sharded_1d):
    """End to end through the public API on host buffers: H2D + scan + D2H
    inside the timed region, blocking per step, max over ranks.  Returns
    (pinned, pageable)."""
    import torch

    import paper_2312_14874_b200 as ps

    rows = cfg.get("rows")
    exclusive = cfg["exclusive"]
    n_local = x.numel()
    sample = n_local if world == 1 else min(n_local, E2E_SAMPLE_MAX)
    if world == 1 and x_host is not None:
        hin = x_host
    else:
        flat = x.reshape(-1)[:sample] if not rows else x[: max(1, sample // cfg["cols"])]
        hin = flat.cpu().numpy()
        sample = hin.size
    hout = np.zeros(hin.shape, np.dtype(cfg["dout"]))
    steps = max(2, min(args.steps, args.e2e_steps))

    if world == 1 and not sharded_1d:
        if rows:
            def step():  # per-row scans of host rows: ps_scan_batched_host pipeline, blocking
                device.scan_batched_host(hin, hout, exclusive=exclusive)
            api = "paper_2312_14874_b200.device.scan_batched_host (ps_scan_batched_host)"
        else:
            def step():  # the drop-in: core.scan_into -> ps_scan_host pipeline, blocking
                ps.core.scan_into(hin, hout, ps.full_span(hin), 0, exclusive=exclusive)
            api = "paper_2312_14874_b200.core.scan_into (ps_scan_host)"
    else:
        sharded = make_sharded(scheme, args.exchange, world)[0] if not rows else None
        dx = torch.empty(hin.shape, dtype=x.dtype, device=dev_t)
        dout = torch.empty(hin.shape, dtype=out.dtype, device=dev_t)
        tin, tout = torch.from_numpy(hin), torch.from_numpy(hout)

        def step():
            dx.copy_(tin, non_blocking=True)
            if rows:
                device.scan_batched(dx, dout, exclusive=exclusive)
            else:
                sharded(dx, dout, exclusive=exclusive, want_total=False)
            tout.copy_(dout, non_blocking=True)
            torch.cuda.current_stream().synchronize()
        api = "H2D copy + device API (ShardedScan / scan_batched) + D2H copy"

    def timed():
        step()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(steps):
            step()
        el = time.perf_counter() - t0
        el = max_over_ranks(el, dist, world, dev_t)
        return {"value": sample * world * steps / el, "unit": "elements/s",
                "h2d_bytes_per_step": hin.nbytes * world, "d2h_bytes_per_step": hout.nbytes * world,
                "steps": steps, "api": api,
                "sample": "the whole job" if sample == n_local else f"{sample} elements per rank"}

    pageable = timed()
    pageable["host_memory"] = ("pageable numpy arrays (the reference's calling convention), staged through the "
                               "library's pinned bounce ring by host copy threads")
    t0 = time.perf_counter()
    with device.pinned_host(hin, hout):
        reg_s = time.perf_counter() - t0
        pinned = timed()
    pinned["host_memory"] = "the same arrays page-locked in place (device.pinned_host -> cudaHostRegister)"
    pinned["register_s"] = reg_s  # one-time cost of page-locking both arrays, outside the timed steps
    return pinned, pageable


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="cfg5")
    ap.add_argument("--scaling", choices=("weak", "strong"), default="weak",
                    help="N>1: weak = every GPU scans a config-sized shard; strong = the config's n split "
                         "across the GPUs (EQUAL layout)")
    ap.add_argument("--scheme", choices=("accumulate-scan", "scan-increment"), default="accumulate-scan")
    ap.add_argument("--exchange", choices=("p2p", "nccl"), default="p2p",
                    help="N>1: shard totals through peer-memory mailboxes inside the kernels (p2p, falls back "
                         "to nccl if unavailable) or one NCCL all-gather between the passes")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--force-sharded", action="store_true",
                    help="use the multi-GPU ShardedScan path even on one GPU (reduce + exchange + carry-in)")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        args.warmup = 3  # timing rule: at least 3 warm-up steps
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
        return 0
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return launch_ranks(args.gpus, os.path.abspath(__file__), sys.argv[1:] if argv is None else list(argv))
    run_ours(args, cfg, args.config)
    return 0


if __name__ == "__main__":
    sys.exit(main())
