#!/usr/bin/env python
"""Top stalled SASS instructions of one kernel in an ncu report.
usage: ncu_source_top.py REPORT KERNEL_REGEX [N]"""
import csv, io, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 15
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kre}", "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
hdr = rows[hi]
ai, si = hdr.index("Address"), hdr.index("Source")
wi, ei = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
data = []
for r in rows[hi + 1:]:
    if len(r) <= max(wi, ei):
        continue
    try:
        data.append((int(r[wi] or 0), r[ai][-5:], r[si].strip(), int(r[ei] or 0)))
    except ValueError:
        pass
print("samples", sum(d[0] for d in data), "warp-instructions executed", sum(d[3] for d in data))
for d in sorted(data, reverse=True)[:n]:
    print(d)
