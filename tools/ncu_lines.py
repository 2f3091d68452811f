#!/usr/bin/env python
"""Aggregate ncu warp-stall samples and executed instructions per CUDA source line.
usage: ncu_lines.py REPORT KERNEL_REGEX [N]"""
import csv, io, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kre}", "--launch-count", "1",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
cur, agg, hdr = None, {}, None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or r[2] != "-":
        continue
    try:
        agg[(cur, int(r[0]))] = (int(r[4] or 0), int(r[7] or 0), r[1].strip()[:100])
    except ValueError:
        pass
tot = sum(v[0] for v in agg.values())
ti = sum(v[1] for v in agg.values())
print(f"samples {tot}  warp-instructions {ti}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"{k[0]}:{k[1]:<5} {v[0]:6d} {100 * v[0] / max(tot, 1):5.1f}%  instr {v[1]:9d}  {v[2]}")
