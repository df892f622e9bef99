"""SASS evidence per production kernel of libprefixscan_b200.so:

    python scripts/sass_summary.py [out.md]

For every kernel instantiation (stall-injection builds excluded): registers,
spill stores/loads and stack from `nvcc -Xptxas -v`, and counts of the SASS
that carries the data path -- UBLKCP (TMA bulk copy), SYNCS (mbarrier),
LDG/STG ...256 (256-bit global accesses), LDS/STS, LDL/STL (local memory:
must be 0), SHFL, REDUX, F2F (float<->double conversions, XU pipe)."""
import os
import re
import subprocess
import sys
from collections import Counter, defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "paper_2312_14874_b200", "csrc", "prefixscan_b200.cu")
LIB = os.path.join(ROOT, "paper_2312_14874_b200", "libprefixscan_b200.so")
PATTERNS = {
    "UBLKCP": r"\bUBLKCP", "SYNCS": r"\bSYNCS\.", "LDG.256": r"\bLDG\.[A-Z0-9.]*256", "STG.256": r"\bSTG\.[A-Z0-9.]*256",
    "LDS": r"\bLDS\b|\bLDS\.", "STS": r"\bSTS\b|\bSTS\.", "LDL/STL": r"\bLDL\b|\bSTL\b|\bLDL\.|\bSTL\.",
    "SHFL": r"\bSHFL\.", "REDUX": r"\bREDUX", "F2F": r"\bF2F\.",
}


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
    return dict(zip(names, out))


def ptxas_info():
    cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-Xptxas", "-v", "-shared",
           "-Xcompiler", "-fPIC", "-o", "/tmp/_sass_summary.so", SRC]
    err = subprocess.run(cmd, capture_output=True, text=True).stderr
    info, cur = {}, None
    for ln in err.splitlines():
        m = re.search(r"Compiling entry function '([^']+)'", ln) or re.search(r"Function properties for (\S+)", ln)
        if m:
            cur = m.group(1)
            info.setdefault(cur, {})
        m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", ln)
        if m and cur:
            info[cur].update(stack=int(m.group(1)), spill_st=int(m.group(2)), spill_ld=int(m.group(3)))
        m = re.search(r"Used (\d+) registers", ln)
        if m and cur:
            info[cur]["regs"] = int(m.group(1))
    return info


def sass_counts():
    txt = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    counts, cur = defaultdict(Counter), None
    for ln in txt.splitlines():
        m = re.search(r"Function : (\S+)", ln)
        if m:
            cur = m.group(1)
            continue
        if cur and "/*" in ln:
            for k, p in PATTERNS.items():
                if re.search(p, ln):
                    counts[cur][k] += 1
    return counts


def main():
    out_path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "r02_sass.md")
    info = ptxas_info()
    counts = sass_counts()
    names = sorted(set(info) | set(counts))
    dem = demangle(names)
    rows = []
    for n in names:
        d = dem.get(n, n)
        # stall-injection instantiations (the STALL template argument) are not production kernels
        m = re.search(r"(scan_stream_kernel|scan_rounds_kernel|scan_rows_kernel|scan_rows_multi_kernel)<([^>]*)>", d)
        if m:
            args = [x.strip() for x in m.group(2).split(",")]
            stall_at = {"scan_stream_kernel": 6, "scan_rounds_kernel": 8, "scan_rows_kernel": 7,
                        "scan_rows_multi_kernel": 7}[m.group(1)]
            if len(args) > stall_at and args[stall_at] == "true":
                continue
        c, i = counts.get(n, Counter()), info.get(n, {})
        rows.append((d.split("(")[0][:110], i.get("regs", "?"), i.get("spill_st", "?"), i.get("spill_ld", "?"),
                     i.get("stack", "?"), *[c[k] for k in PATTERNS]))
    lines = ["# SASS evidence per production kernel (`python scripts/sass_summary.py`)", "",
             "Registers / spills / stack from `nvcc -Xptxas -v`; opcode counts from `cuobjdump -sass` of "
             "the built library (static counts per kernel).  Stall-injection builds are excluded.", "",
             "| kernel | regs | spill st | spill ld | stack | " + " | ".join(PATTERNS) + " |",
             "|---|" + "---|" * (4 + len(PATTERNS))]
    for r in rows:
        lines.append("| `" + r[0] + "` | " + " | ".join(str(v) for v in r[1:]) + " |")
    spills = [r for r in rows if r[2] not in (0, "?") or r[3] not in (0, "?")]
    lines += ["", f"{len(rows)} kernels; {len(spills)} with spills."]
    open(out_path, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines[-3:]))


if __name__ == "__main__":
    main()
