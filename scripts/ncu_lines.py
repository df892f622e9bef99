"""Per-CUDA-source-line stall samples / instructions from an ncu report (dev tool).
usage: python scripts/ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
cur, hdr, out = None, None, []
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) >= len(hdr) - 1 and r[2] == "-":
        try:
            s = int(r[4]); ie = int(r[7])
        except ValueError:
            continue
        stalls = {hdr[i]: int(r[i]) for i in range(len(hdr)) if hdr[i].startswith("stall_") and "(" not in hdr[i]
                  and r[i].isdigit() and int(r[i]) > 0}
        out.append((s, ie, cur, r[0], r[1].strip()[:60], stalls))
tot_s = sum(o[0] for o in out); tot_i = sum(o[1] for o in out)
print(f"samples {tot_s}  warp-instructions {tot_i}")
for o in sorted(out, key=lambda x: -x[0])[:top]:
    st = " ".join(f"{k[6:]}={v}" for k, v in sorted(o[5].items(), key=lambda kv: -kv[1])[:3])
    print(f"{o[0]:6d} {o[1]:10d} {o[2]}:{o[3]:<4} {o[4]:<60} {st}")
print("--- by instructions")
for o in sorted(out, key=lambda x: -x[1])[:top]:
    print(f"{o[1]:10d} {o[2]}:{o[3]:<4} {o[4]}")
