"""Attribute an ncu source-page capture (SASS, per instruction) to CUDA source
lines through the cubin's line table:

    python scripts/ncu_lines.py <ncu-source.csv> <nvdisasm -g output> <kernel mangled name>

Prints issued instructions and warp-stall samples per file:line, largest first."""
import csv
import re
import sys
from collections import defaultdict

src_csv, sass, kname = sys.argv[1:4]
# offset -> (file, line) from nvdisasm -g
lines = {}
cur = None
inside = False
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
agg = defaultdict(lambda: [0, 0, 0])
for r in body:
    off = int(r[col["Address"]], 16) - base
    key = lines.get(off, ("?", 0))
    agg[key][0] += int(r[col["Instructions Executed"]] or 0)
    agg[key][1] += int(r[col["Warp Stall Sampling (All Samples)"]] or 0)
    agg[key][2] += int(r[col["Warp Stall Sampling (Not-issued Samples)"]] or 0)
tot = [sum(v[i] for v in agg.values()) for i in range(3)]
print(f"total: {tot[0]} warp instructions, {tot[1]} stall samples")
for key, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:int(sys.argv[4]) if len(sys.argv) > 4 else 40]:
    print(f"{key[0]}:{key[1]:<5d} inst {v[0]:>11d} ({100*v[0]/tot[0]:5.1f}%)  samples {v[1]:>7d} ({100*v[1]/tot[1]:5.1f}%)"
          f"  not-issued {v[2]:>7d}")
