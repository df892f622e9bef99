"""Per-SASS-instruction view of an ncu source-page CSV joined with the cubin's line table:
    python scripts/ncu_hot.py <source.csv> <nvdisasm -g output> <mangled kernel> [min executions]
prints address, executions, stall samples, file:line and the instruction."""
import csv
import re
import sys

src_csv, sass, kname = sys.argv[1:4]
thr = int(sys.argv[4]) if len(sys.argv) > 4 else 1
lines, cur, inside = {}, None, False
for ln in open(sass):
    if ln.startswith(".text."):
        inside = ln.strip() == f".text.{kname}:"
        continue
    if not inside:
        continue
    m = re.search(r'//## File "(.*)", line (\d+)', ln)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
    if m and cur:
        lines[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(src_csv)))
head = rows[1]
col = {k: i for i, k in enumerate(head)}
body = [r for r in rows[2:] if len(r) == len(head)]
base = int(body[0][col["Address"]], 16)
for r in body:
    off = int(r[col["Address"]], 16) - base
    n = int(r[col["Instructions Executed"]] or 0)
    if n >= thr:
        f, l = lines.get(off, ("?", 0))
        print(f'{off:05x} {n:>9d} {r[col["Warp Stall Sampling (All Samples)"]]:>5s} {f}:{l:<4d} {r[col["Source"]][:80]}')
