"""Turn ncu outputs from gpurun_out/ into committed summaries under profiles/.

    python scripts/summarize_ncu.py <tag> <config> <launches.csv> [<full.ncu-rep>]

* launches.csv  -- `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
                   dram__bytes_write.sum --csv --log-file ...` of a bench run
* full.ncu-rep  -- `ncu --set full` capture of the dominant kernel
Writes profiles/<tag>_<config>_launches.md and, with a capture,
profiles/<tag>_<config>_full.md, and updates profiles/traffic.json with the
per-launch DRAM bytes of the dominant (scan) kernel for bench.py.
"""

import csv
import json
import os
import statistics
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

FULL_METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    head, body = rows[0], rows[1:]
    col = {k: i for i, k in enumerate(head)}
    per = defaultdict(lambda: defaultdict(dict))
    for r in body:
        per[r[col["Kernel Name"]]][r[col["ID"]]][r[col["Metric Name"]]] = float(r[col["Metric Value"]])
    return per


def main():
    tag, cfg, lpath = sys.argv[1:4]
    full = sys.argv[4] if len(sys.argv) > 4 else None
    os.makedirs(PROF, exist_ok=True)
    per = launches(lpath)
    lines = [f"# {tag} {cfg}: ncu launch list (`--metrics gpu__time_duration.sum,dram__bytes_read.sum,"
             f"dram__bytes_write.sum --clock-control none`)", "",
             "Per-launch times are cold-cache and serialised under ncu: compare shares, not absolutes.", "",
             "| kernel | launches | mean time (us) | share of GPU time | DRAM read/launch (MB) | DRAM write/launch (MB) |",
             "|---|---|---|---|---|---|"]
    total = sum(m.get("gpu__time_duration.sum", 0) for k in per for m in per[k].values())
    dominant, dom_time = None, -1.0
    for k, ids in sorted(per.items(), key=lambda kv: -sum(m.get("gpu__time_duration.sum", 0) for m in kv[1].values())):
        ts = [m.get("gpu__time_duration.sum", 0) for m in ids.values()]
        rd = [m.get("dram__bytes_read.sum", 0) for m in ids.values()]
        wr = [m.get("dram__bytes_write.sum", 0) for m in ids.values()]
        t = sum(ts)
        lines.append(f"| `{k[:90]}` | {len(ts)} | {statistics.mean(ts) / 1e3:.1f} | {100 * t / total:.1f}% | "
                     f"{statistics.mean(rd) / 1e6:.1f} | {statistics.mean(wr) / 1e6:.1f} |")
        if t > dom_time:
            dominant, dom_time = k, t
    ids = per[dominant]
    traffic = statistics.mean(m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
                              for m in ids.values())
    lines += ["", f"Dominant kernel: `{dominant}`; DRAM traffic per launch {traffic / 1e9:.4f} GB."]
    open(os.path.join(PROF, f"{tag}_{cfg}_launches.md"), "w").write("\n".join(lines) + "\n")
    tj = os.path.join(PROF, "traffic.json")
    data = json.load(open(tj)) if os.path.exists(tj) else {}
    data[cfg] = {"dram_bytes_per_launch": traffic, "kernel": dominant, "source": f"profiles/{tag}_{cfg}_launches.md"}
    json.dump(data, open(tj, "w"), indent=1)
    if full:
        if full.endswith(".csv"):  # already exported on the GPU box (`ncu -i x.ncu-rep --page raw --csv`)
            raw = open(full).read()
        else:
            raw = subprocess.run(["ncu", "-i", full, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(raw.splitlines()))
        head, units, vals = rows[0], rows[1], rows[2]
        out = [f"# {tag} {cfg}: `ncu --set full` of `{vals[head.index('Kernel Name')]}`", "",
               "| metric | unit | value |", "|---|---|---|"]
        for m in FULL_METRICS:
            if m in head:
                i = head.index(m)
                out.append(f"| {m} | {units[i]} | {vals[i]} |")
        open(os.path.join(PROF, f"{tag}_{cfg}_full.md"), "w").write("\n".join(out) + "\n")
    print(f"dominant {dominant}: traffic/launch {traffic:.0f} B")


if __name__ == "__main__":
    main()
